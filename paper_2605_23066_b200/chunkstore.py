"""Chunked n-d arrays: grid rules, the native chunk writer/reader, metadata merge.

On-disk format (identical to the reference, ``chunkstore.py:1-14``): an array is a grid
of write chunks aligned to shard boundaries, optionally subdivided into read chunks;
a chunk payload is the raw little-endian row-major bytes of its box.  Two layouts:

* per-leaf   — one object ``<prefix>/<leaf>/c.<i0>.<i1>…`` per write chunk;
* aggregated — payloads appended to ``<prefix>/d/<file_id>`` data files (greedy flush when
  the next payload would exceed the target), located through ``manifest.json``.

What is B200-specific: chunk payloads are never materialised by Python.
``ProcessArrayWriter`` turns every chunk into a descriptor (source device address, box,
output file, offset) and the native engine packs strided boxes on the GPU, DMA's them
into pinned slots and writes them with its own threads; ``ChunkReader.read_range`` and
the load pipeline do the inverse.  The grid arithmetic, key names, manifest and metadata
documents are host logic mirroring ``chunkstore.py:50-246, 249-305, 426-454, 603-690``.
"""

from __future__ import annotations

import bisect
import functools
import itertools
import math
import re
from bisect import bisect_left
from dataclasses import dataclass, field
from typing import Any, Iterable, Iterator, Optional, Sequence

import numpy as np

from . import docio
from .backend import Store
from .dtypes import itemsize, numpy_dtype
from .errors import (
    AlignmentError,
    ChunkStoreError,
    ConsistencyError,
    CorruptionError,
    DuplicateChunkError,
    MissingKeyError,
)
from .sharding import Range, segment_axis

PER_LEAF = "per_leaf"
AGGREGATED = "aggregated"
LAYOUTS = (PER_LEAF, AGGREGATED)

DEFAULT_TARGET_FILE_BYTES = 64 * 1024 * 1024

ARRAY_METADATA_FILE = "array_metadata.json"
MANIFEST_FILE = "manifest.json"
DATA_DIR = "d"


def _divides(part: int, whole: int) -> bool:
    if whole == 0:
        return part == 0
    return part >= 1 and whole % part == 0


@dataclass(frozen=True)
class ChunkGrid:
    """Write-chunk and read-subchunk shapes over one shard grid."""

    shard_shape: tuple[int, ...]
    write_chunk: tuple[int, ...]
    read_chunk: tuple[int, ...]

    def __post_init__(self):
        for s, w, r in zip(self.shard_shape, self.write_chunk, self.read_chunk):
            if not _divides(w, s):
                raise ChunkStoreError(
                    f"write chunk {self.write_chunk} does not subdivide shard {self.shard_shape}"
                )
            if not _divides(r, w):
                raise ChunkStoreError(
                    f"read chunk {self.read_chunk} does not subdivide write chunk {self.write_chunk}"
                )


@dataclass(frozen=True)
class ArrayStorageMetadata:
    global_shape: tuple[int, ...]
    dtype: str
    shard_shape: tuple[int, ...]
    write_chunk: tuple[int, ...]
    read_chunk: tuple[int, ...]
    layout: str

    def __post_init__(self):
        if self.layout not in LAYOUTS:
            raise ChunkStoreError(f"unknown layout {self.layout!r}")
        if not _grid_consistent(self.global_shape, self.shard_shape):
            raise ChunkStoreError(
                f"shard {self.shard_shape} does not subdivide global {self.global_shape}"
            )
        ChunkGrid(self.shard_shape, self.write_chunk, self.read_chunk)
        numpy_dtype(self.dtype)

    @property
    def rank(self) -> int:
        return len(self.global_shape)

    def chunk_counts(self) -> tuple[int, ...]:
        return tuple(0 if g == 0 else g // w for g, w in zip(self.global_shape, self.write_chunk))

    def total_chunks(self) -> int:
        return math.prod(self.chunk_counts())

    def chunk_nbytes(self) -> int:
        return math.prod(self.write_chunk) * itemsize(self.dtype)

    def to_json(self) -> dict:
        return {
            "global_shape": list(self.global_shape),
            "dtype": self.dtype,
            "shard_shape": list(self.shard_shape),
            "write_chunk": list(self.write_chunk),
            "read_chunk": list(self.read_chunk),
            "layout": self.layout,
        }

    @classmethod
    def from_json(cls, doc: dict) -> "ArrayStorageMetadata":
        try:
            key = (tuple(doc["global_shape"]), doc["dtype"], tuple(doc["shard_shape"]),
                   tuple(doc["write_chunk"]), tuple(doc["read_chunk"]), doc["layout"])
            return _storage_meta_of(*key)  # leaves share a handful of distinct entries
        except (KeyError, TypeError) as exc:
            raise CorruptionError(f"malformed array metadata: {exc}") from exc


@functools.lru_cache(maxsize=1 << 14)
def _storage_meta_of(*key) -> ArrayStorageMetadata:
    return ArrayStorageMetadata(*key)


def _grid_consistent(global_shape: tuple[int, ...], part: tuple[int, ...]) -> bool:
    return len(part) == len(global_shape) and all(
        _divides(p, g) for p, g in zip(part, global_shape)
    )


def _smallest_prime_factor(n: int) -> int:
    if n % 2 == 0:
        return 2
    f = 3
    while f * f <= n:
        if n % f == 0:
            return f
        f += 2
    return n


def choose_chunk_shape(shard_shape: tuple[int, ...], dtype: str, target_bytes: int) -> tuple[int, ...]:
    """Read-chunk shape dividing ``shard_shape`` with at most ``target_bytes`` per chunk
    when reachable.  Dims are reduced largest-first (ties: lowest index), halving while
    even, else dividing by the smallest prime factor (``chunkstore.py:156-182``)."""
    isz = itemsize(dtype)
    if target_bytes < isz:
        raise ChunkStoreError(f"target {target_bytes} B below element size {isz} B")
    chunk = [int(s) for s in shard_shape]
    if 0 in chunk:
        return tuple(chunk)
    for d in sorted(range(len(chunk)), key=lambda i: (-shard_shape[i], i)):
        while chunk[d] > 1 and math.prod(chunk) * isz > target_bytes:
            chunk[d] //= 2 if chunk[d] % 2 == 0 else _smallest_prime_factor(chunk[d])
    return tuple(chunk)


def derive_write_chunk(shard_shape: tuple[int, ...], n_segments: int) -> tuple[int, ...]:
    """Write chunk aligned with ceil-division replica segmenting: the segment axis extent
    becomes gcd(ceil(s/n), s) (``chunkstore.py:185-202``)."""
    if n_segments <= 1 or not shard_shape or 0 in shard_shape:
        return tuple(shard_shape)
    axis = segment_axis(tuple(shard_shape))
    s = shard_shape[axis]
    chunk = list(shard_shape)
    chunk[axis] = math.gcd(-(-s // n_segments), s)
    return tuple(chunk)


def coords_key(coords: tuple[int, ...]) -> str:
    return ".".join(map(str, coords)) if coords else "0"


def chunk_object_key(leaf_path: str, coords: tuple[int, ...]) -> str:
    return f"{leaf_path}/c.{coords_key(coords)}"


def _covering(ranges: tuple[Range, ...], steps: tuple[int, ...]) -> Iterator[tuple[int, ...]]:
    """Grid coordinates (product order) of the cells meeting ``ranges``."""
    spans = []
    for (off, ext), step in zip(ranges, steps):
        if ext == 0:
            return
        spans.append(range(off // step, (off + ext - 1) // step + 1))
    yield from itertools.product(*spans)


def _cell_ranges(coords: tuple[int, ...], steps: tuple[int, ...]) -> tuple[Range, ...]:
    return tuple((c * s, s) for c, s in zip(coords, steps))


def _intersect(a: tuple[Range, ...], b: tuple[Range, ...]) -> tuple[Range, ...] | None:
    out = []
    for (ao, ae), (bo, be) in zip(a, b):
        lo, hi = max(ao, bo), min(ao + ae, bo + be)
        if lo >= hi:
            return None
        out.append((lo, hi - lo))
    return tuple(out)


def _slab_is_contiguous(extents: tuple[int, ...], shape: tuple[int, ...]) -> bool:
    """Is a leading box of ``extents`` one contiguous run inside ``shape``?"""
    partial = [d for d, (e, s) in enumerate(zip(extents, shape)) if e != s]
    if not partial:
        return True
    return all(extents[d] == 1 for d in range(partial[-1]))


def _strides(shape: tuple[int, ...]) -> tuple[int, ...]:
    out = [1] * len(shape)
    for d in range(len(shape) - 2, -1, -1):
        out[d] = out[d + 1] * shape[d + 1]
    return tuple(out)


class BoxIndex:
    """Which of a set of boxes meet a query box, without testing every box.

    Target shardings are grids (mesh axes split dimensions), so per dimension the boxes'
    intervals are either identical or disjoint: a query is answered by a bisection per
    dimension and a lookup of the product of the intervals it meets.  Any other set of
    boxes falls back to the linear scan.  Results keep the input order."""

    def __init__(self, boxes: Sequence[tuple[Range, ...]]):
        self.boxes = [tuple(b) for b in boxes]
        self.by_box: dict[tuple[Range, ...], list[int]] = {}
        for i, b in enumerate(self.boxes):
            self.by_box.setdefault(b, []).append(i)
        rank = len(self.boxes[0]) if self.boxes else 0
        self.dims: list[list[Range]] | None = []
        for d in range(rank):
            iv = sorted({b[d] for b in self.boxes})
            if any(o1 + e1 > o2 for (o1, e1), (o2, _) in zip(iv, iv[1:])):
                self.dims = None  # overlapping intervals: not a grid
                break
            self.dims.append(iv)
        if self.dims is not None and math.prod(len(iv) for iv in self.dims) != len(self.by_box):
            self.dims = None      # not every product cell is a box: not a full grid

    def hits(self, box: tuple[Range, ...]) -> list[int]:
        if self.dims is None:
            return [i for i, b in enumerate(self.boxes) if _intersect(box, b) is not None]
        per_dim = []
        for (bo, be), iv in zip(box, self.dims):
            lo = bisect.bisect_right(iv, (bo, math.inf)) - 1
            lo = max(lo, 0)
            sel = []
            for j in range(lo, len(iv)):
                o, e = iv[j]
                if o >= bo + be:
                    break
                if o + e > bo and e > 0 and be > 0:
                    sel.append(iv[j])
            if not sel:
                return []
            per_dim.append(sel)
        out: list[int] = []
        for cell in itertools.product(*per_dim):
            out.extend(self.by_box.get(cell, ()))
        out.sort()
        return out


def box_is_contiguous(shape: Sequence[int], off: Sequence[int], ext: Sequence[int]) -> bool:
    """Is box (off, ext) a single byte run of a row-major array of ``shape``?"""
    dims = [d for d, e in enumerate(ext) if e > 1]
    if not dims:
        return True
    return all(ext[d] == shape[d] for d in range(dims[0] + 1, len(shape)))


def box_flat_offset(shape: Sequence[int], off: Sequence[int]) -> int:
    return sum(o * s for o, s in zip(off, _strides(tuple(shape))))


class AggregatedManifest:
    """Sorted chunk key -> (file_id, offset, length) index of aggregated data files."""

    def __init__(self, entries: dict[str, tuple[int, int, int]], target_file_bytes: int):
        self._keys = sorted(entries)
        self._locs = [tuple(entries[k]) for k in self._keys]
        self.target_file_bytes = target_file_bytes
        self._validate()

    def _validate(self) -> None:
        spans: dict[int, list[tuple[int, int]]] = {}
        for fid, off, length in self._locs:
            if off < 0 or length < 0:
                raise CorruptionError("negative manifest byte range")
            spans.setdefault(fid, []).append((off, length))
        for fid, ranges in spans.items():
            ranges.sort()
            for (o1, l1), (o2, _) in zip(ranges, ranges[1:]):
                if o1 + l1 > o2:
                    raise CorruptionError(f"overlapping byte ranges in data file {fid}")

    def __len__(self) -> int:
        return len(self._keys)

    def keys(self) -> list[str]:
        return list(self._keys)

    def lookup(self, key: str) -> tuple[int, int, int]:
        i = bisect_left(self._keys, key)
        if i == len(self._keys) or self._keys[i] != key:
            raise MissingKeyError(f"chunk key {key!r} not in manifest")
        return self._locs[i]

    def to_json(self) -> dict:
        return {
            "target_file_bytes": self.target_file_bytes,
            "entries": {k: list(v) for k, v in zip(self._keys, self._locs)},
        }

    @classmethod
    def from_json(cls, doc: dict) -> "AggregatedManifest":
        try:
            entries = {k: (int(f), int(o), int(l)) for k, (f, o, l) in doc["entries"].items()}
            return cls(entries, int(doc["target_file_bytes"]))
        except (KeyError, TypeError, ValueError) as exc:
            raise CorruptionError(f"malformed manifest: {exc}") from exc


# -- device regions ---------------------------------------------------------------------


@dataclass(slots=True)
class DeviceRegion:
    """Where the values of one box live on a GPU: the contiguous row-major array at
    ``address`` of extents ``shape`` holds the box at offset ``origin``.  A shard, a
    global array and a slice of a packed snapshot arena are all DeviceRegions — no copy
    (and no tensor view) is made to describe a box.  ``owner`` keeps the memory alive."""

    address: int
    shape: tuple[int, ...]
    origin: tuple[int, ...]
    gpu: int
    owner: Any = None

    @classmethod
    def of(cls, tensor, origin: tuple[int, ...]) -> "DeviceRegion":
        return cls(int(tensor.data_ptr()), tuple(int(s) for s in tensor.shape), tuple(origin),
                   tensor.device.index, tensor)


def as_device_region(values: Any, extents: tuple[int, ...], dtype: str, gpu: int | None = None) -> DeviceRegion:
    """Accept a DeviceRegion, a torch CUDA tensor of exactly ``extents`` or a host numpy
    array (uploaded once — the compatibility path of ``write_array`` callers that pass
    numpy boxes)."""
    import torch

    from .dtypes import torch_dtype

    if isinstance(values, DeviceRegion):
        return values
    if isinstance(values, torch.Tensor):
        t = values
        if not t.is_cuda:
            dev = torch.device("cuda", gpu if gpu is not None else torch.cuda.current_device())
            t = t.to(dev)
    else:
        from .treemodel import _host_storage

        host = np.asarray(_host_storage(values, dtype), order="C")  # keeps 0-d arrays 0-d
        dev = torch.device("cuda", gpu if gpu is not None else torch.cuda.current_device())
        t = torch.from_numpy(host.reshape(-1).view(np.uint8)).to(dev)
        t = t.view(torch_dtype(dtype)).reshape(host.shape) if host.size else torch.empty(
            host.shape, dtype=torch_dtype(dtype), device=dev)
    if tuple(t.shape) != tuple(extents):
        raise AlignmentError(f"shard buffer shape {tuple(t.shape)} does not match extents {extents}")
    t = t.contiguous()
    return DeviceRegion.of(t, (0,) * len(extents))


def _fill_box(rec: np.ndarray, base: int, shape: Sequence[int], off: Sequence[int]) -> None:
    rec["base"] = base
    rank = len(shape)
    rec["shape"][:rank] = shape
    rec["off"][:rank] = off


# -- writer ---------------------------------------------------------------------------------


@dataclass(slots=True)
class _PendingChunk:
    key: str          # full storage key of the output (chunk object, or data file)
    region: DeviceRegion
    box_off: tuple[int, ...]   # chunk origin inside region.tensor
    ext: tuple[int, ...]
    itemsize: int
    nbytes: int
    file_off: int


class ProcessArrayWriter:
    """Writes one process's chunks under ``<prefix>`` (``chunkstore.py:307-454``).

    ``write_array`` plans (keys, file offsets, duplicate checks); the bytes move in
    ``flush`` — one native engine call for everything pending.  The save pipeline
    builds its writer ``deferred``: every array of the process goes in ONE engine call
    at ``finish`` (which then writes the manifest and ``array_metadata.json``).  A
    writer used directly (``deferred=False``, the default) stores each array's chunks
    before ``write_array`` returns, like the reference (aggregated: the data files that
    are complete; the open one at ``finish``).  Op order on the backend is the
    reference's: chunk puts in write order, then manifest, then metadata.
    """

    def __init__(self, store: Store, prefix: str, layout: str,
                 target_file_bytes: int = DEFAULT_TARGET_FILE_BYTES, *, engine_cfg=None,
                 concurrent: int = 1, deferred: bool = False):
        if layout not in LAYOUTS:
            raise ChunkStoreError(f"unknown layout {layout!r}")
        self._store = store
        self._prefix = prefix.rstrip("/")
        self._layout = layout
        self._target = target_file_bytes
        self._metas: dict[str, ArrayStorageMetadata] = {}
        self._shardings: dict[str, Optional[dict]] = {}
        self._chunks: dict[str, set[str]] = {}
        self._manifest_entries: dict[str, tuple[int, int, int]] = {}
        self._pending: list[_PendingChunk] = []
        self._fid = 0        # aggregated: current data file id
        self._cur_fill = 0   # aggregated: bytes already assigned to it
        self._finished = False
        self._engine_cfg = engine_cfg
        self._concurrent = concurrent
        self._deferred = deferred
        self.stats = None

    def declare_array(self, leaf_path: str, meta: ArrayStorageMetadata,
                      sharding_descriptor: dict | None = None) -> None:
        if meta.layout != self._layout:
            raise ChunkStoreError("array layout differs from writer layout")
        known = self._metas.get(leaf_path)
        if known is not None and known != meta:
            raise ConsistencyError(f"conflicting metadata for {leaf_path!r}")
        self._metas[leaf_path] = meta
        self._shardings.setdefault(leaf_path, sharding_descriptor)
        self._chunks.setdefault(leaf_path, set())

    def write_array(self, leaf_path: str, shards: Iterable[tuple[tuple[Range, ...], Any]],
                    meta: ArrayStorageMetadata, sharding_descriptor: dict | None = None) -> list[str]:
        """Plan whole write chunks of each (ranges, values) piece; returns the keys the
        chunks will be stored under.  ``values`` is a DeviceRegion / CUDA tensor / numpy
        box exactly covering ``ranges``."""
        self.declare_array(leaf_path, meta, sharding_descriptor)
        isz = itemsize(meta.dtype)
        keys = []
        for ranges, values in shards:
            ranges = tuple((int(o), int(e)) for o, e in ranges)
            if len(ranges) != meta.rank:
                raise AlignmentError(f"rank mismatch for {leaf_path!r}")
            for (off, ext), w, g in zip(ranges, meta.write_chunk, meta.global_shape):
                if off < 0 or off + ext > g:
                    raise AlignmentError(
                        f"range ({off}, {ext}) outside global extent {g} for {leaf_path!r}"
                    )
                if ext and (off % w or ext % w):
                    raise AlignmentError(
                        f"range ({off}, {ext}) of {leaf_path!r} not aligned to write chunk "
                        f"{meta.write_chunk}"
                    )
            extents = tuple(e for _, e in ranges)
            region = as_device_region(values, extents, meta.dtype)
            if not isinstance(values, DeviceRegion) and region.shape != extents:
                raise AlignmentError(
                    f"shard buffer shape {region.shape} does not match ranges {ranges} "
                    f"for {leaf_path!r}"
                )
            nbytes = math.prod(meta.write_chunk) * isz
            for coords in _covering(ranges, meta.write_chunk):
                box_off = tuple(
                    o + c * w - r0
                    for o, c, w, (r0, _) in zip(region.origin, coords, meta.write_chunk, ranges)
                )
                keys.append(self._plan_chunk(leaf_path, coords, region, box_off, meta.write_chunk,
                                             isz, nbytes))
        if not self._deferred:
            self._flush_complete()
        return keys

    def _flush_complete(self) -> None:
        """Store the pending chunks whose output is complete (per-leaf: all of them;
        aggregated: those of data files before the open one)."""
        if self._layout == PER_LEAF:
            self.flush()
            return
        open_key = f"{self._prefix}/{DATA_DIR}/{self._fid}"
        done = [p for p in self._pending if p.key != open_key]
        if done:
            self._pending = [p for p in self._pending if p.key == open_key]
            self.stats = execute_writes(self._store, done, self._engine_cfg, self._concurrent)

    def _plan_chunk(self, leaf_path, coords, region, box_off, ext, isz, nbytes) -> str:
        ck = coords_key(coords)
        seen = self._chunks[leaf_path]
        if ck in seen:
            raise DuplicateChunkError(f"chunk {ck} of {leaf_path!r} written twice")
        seen.add(ck)
        rel = chunk_object_key(leaf_path, coords)
        if self._layout == PER_LEAF:
            key = f"{self._prefix}/{rel}"
            self._pending.append(_PendingChunk(key, region, box_off, ext, isz, nbytes, 0))
            return key
        # Greedy packing (chunkstore.py:409-417): a new file starts when the current one
        # is non-empty and the payload would push it past the target.
        if self._cur_fill and self._cur_fill + nbytes > self._target:
            self._fid += 1
            self._cur_fill = 0
        fid = self._fid
        self._manifest_entries[rel] = (fid, self._cur_fill, nbytes)
        key = f"{self._prefix}/{DATA_DIR}/{fid}"
        self._pending.append(_PendingChunk(key, region, box_off, ext, isz, nbytes, self._cur_fill))
        self._cur_fill += nbytes
        return key

    # -- execution ---------------------------------------------------------------------------

    def flush(self) -> None:
        """Move every planned chunk to storage (one native engine call)."""
        pending, self._pending = self._pending, []
        if not pending:
            return
        self.stats = execute_writes(self._store, pending, self._engine_cfg, self._concurrent)

    def finish(self) -> dict:
        """Flush chunks, then write the manifest (aggregated) and the per-process
        metadata document; returns the document."""
        if self._finished:
            raise ChunkStoreError("writer already finished")
        self._finished = True
        self.flush()
        if self._layout == AGGREGATED:
            manifest = AggregatedManifest(self._manifest_entries, self._target)
            self._store.put(f"{self._prefix}/{MANIFEST_FILE}", docio.dumps_canonical(manifest.to_json()))
        doc = {
            "format_version": 1,
            "layout": self._layout,
            "arrays": {
                leaf: {
                    **meta.to_json(),
                    "sharding": self._shardings.get(leaf),
                    "chunks": sorted(self._chunks[leaf]),
                }
                for leaf, meta in self._metas.items()
            },
        }
        self._store.put(f"{self._prefix}/{ARRAY_METADATA_FILE}", docio.dumps_canonical(doc))
        return doc


_PROCESS_DIR = re.compile(r"(?:^|/)process_(\d+)/")


def process_of_key(key: str) -> int | None:
    """The logical process whose ``process_<p>/`` directory holds ``key`` (None if none)."""
    m = _PROCESS_DIR.search(key)
    return int(m.group(1)) if m else None


def execute_writes(store: Store, pending: list[_PendingChunk], engine_cfg=None, concurrent: int = 1):
    """Run planned chunk writes through the native engine.

    Outputs are the distinct keys in first-appearance order (one per chunk, or one per
    aggregated data file).  The backend admits the puts in that order (fault plan,
    payload gate), the engine writes them, the backend records them.
    """
    from . import native

    out_keys: list[str] = []
    out_index: dict[str, int] = {}
    sizes: list[int] = []
    for p in pending:
        i = out_index.get(p.key)
        if i is None:
            i = out_index[p.key] = len(out_keys)
            out_keys.append(p.key)
            sizes.append(0)
        sizes[i] = max(sizes[i], p.file_off + p.nbytes)
    backend = store.backend
    store.sched_point()
    n_ok, err = backend.admit_bulk("put", out_keys)
    if n_ok < len(out_keys):
        allowed = set(range(n_ok))
        keep = [p for p in pending if out_index[p.key] in allowed]
        out_keys, sizes = out_keys[:n_ok], sizes[:n_ok]
        pending = keep
    cfg = engine_cfg or native.EngineConfig()
    root = backend.native_root()
    stats = None
    if pending:
        items = native.write_table(
            [p.region.address for p in pending], [p.region.shape for p in pending],
            [p.box_off for p in pending], [p.ext for p in pending], [p.itemsize for p in pending],
            [out_index[p.key] for p in pending], [p.region.gpu for p in pending],
            [p.file_off for p in pending],
        )
        outputs = np.zeros(len(out_keys), native.OUTPUT)
        outputs["size"] = sizes
        host_bufs: list[np.ndarray] = []
        if root is not None:
            paths = native.PathTable([backend.path_of(k) for k in out_keys])
            outputs["path"] = paths.pointers
        else:
            for i, size in enumerate(sizes):
                buf = np.empty(size, np.uint8)
                host_bufs.append(buf)
                outputs[i]["host"] = buf.ctypes.data if size else 0
        pool = backend.recycle_pool(process_of_key(out_keys[0])) if root is not None else None
        # per GPU and save size (rates of a 4 GB and an 80 GB save are not comparable)
        gpu = (int(pending[0].region.gpu), max(1, sum(sizes)).bit_length())
        register = bool(pool) and bool(getattr(backend, "register_pool", False))
        zero_copy = register and native.SAVE_PATHS.choose(gpu)
        with native.engine_lease(cfg, concurrent) as eng:
            stats = eng.save(items, outputs, pool, register=register, zero_copy=zero_copy)
        if pool and int(stats["recycled_files"]) > 0:
            # a save that registered files (once per file lifetime) or, zero-copy, still
            # found unregistered ones is a warm-up: not scored
            warm_up = int(stats["registered_files"]) > 0 or (
                zero_copy and int(stats["zero_copy_bytes"]) < 0.99 * int(stats["bytes_storage"]))
            native.SAVE_PATHS.record(gpu, zero_copy, int(stats["bytes_storage"]), float(stats["seconds_total"]),
                                     warm_up)
        if root is not None:
            backend.record_bulk(store.identity, "put", out_keys, [0] * len(out_keys), sizes)
        else:
            # Non-filesystem backends receive ordinary puts of the produced bytes; the
            # admission above already counted them, so go straight to the backend op.
            for key, buf in zip(out_keys, host_bufs):
                data = buf.tobytes()
                with backend._lock:
                    backend._put(key, data)
                    backend._record(store.identity, "put", key, 0, len(data))
    if err is not None:
        raise err
    return stats


# -- reader -----------------------------------------------------------------------------------


@dataclass
class ReadStats:
    bytes_requested: int = 0
    bytes_loaded: int = 0


@dataclass(slots=True)
class Fetch:
    """One contiguous byte range of a stored chunk and the box it holds."""

    key: str                      # storage key read
    op: str                       # "get" | "get_range"
    file_off: int
    nbytes: int
    origin: tuple[int, ...]       # global origin of the fetched box
    shape: tuple[int, ...]        # box shape (write chunk, read chunk, or a slab of one)
    whole_file: bool
    object_bytes: int = -1        # size a per-leaf chunk object must have (-1: no check)


def plan_fetches(prefix: str, leaf_path: str, entry: dict, meta: ArrayStorageMetadata,
                 requests: Sequence[tuple[Range, ...]]) -> list[Fetch]:
    """Minimal fetch list covering the union of ``requests`` for one array
    (``chunkstore.py:507-578``): per covering write chunk, the whole chunk when every
    subchunk is needed or subchunks are not contiguous in it, else one byte-range fetch
    per needed subchunk."""
    geometry = fetch_geometry(meta.write_chunk, meta.read_chunk, itemsize(meta.dtype),
                              tuple(tuple(r_) for r_ in requests))
    return fetches_at(prefix, leaf_path, entry, geometry)


@functools.lru_cache(maxsize=1 << 12)
def fetch_geometry(w: tuple[int, ...], r: tuple[int, ...], isz: int,
                   requests: tuple[tuple[Range, ...], ...]) -> tuple[tuple, ...]:
    """The storage-independent part of ``plan_fetches``: per fetch ``(chunk coords, chunk
    key, byte offset in the chunk, nbytes, origin, shape, whole chunk, object bytes)``
    where object bytes is the size a per-leaf chunk object read whole must have (-1 for
    subchunk spans).  A pure function of the chunk grid and the requested boxes, so the
    leaves of a tree that share a shape and sharding (every layer of a transformer) share
    one entry."""
    subs_per = tuple(wi // ri for wi, ri in zip(w, r))
    n_subs = math.prod(subs_per)
    contiguous = _slab_is_contiguous(r, w)
    wstrides = _strides(w)
    chunks: dict[tuple[int, ...], set[tuple[int, ...]] | None] = {}
    order: list[tuple[int, ...]] = []
    whole_only = n_subs == 1  # read chunk == write chunk: every covering chunk is read whole
    for ranges in dict.fromkeys(requests):  # replicas ask for the same box
        if any(e == 0 for _, e in ranges):
            continue
        for coords in _covering(ranges, w):
            if whole_only:
                if coords not in chunks:
                    chunks[coords] = None
                    order.append(coords)
                continue
            hit = _intersect(ranges, _cell_ranges(coords, w))
            if hit is None:
                continue
            subs = chunks.get(coords)
            if subs is None:
                subs = chunks[coords] = set()
                order.append(coords)
            subs.update(_covering(hit, r))
    out: list[tuple] = []
    chunk_bytes = math.prod(w) * isz
    sub_bytes = math.prod(r) * isz
    for coords in order:
        ck = coords_key(coords)
        needed = chunks[coords]
        if whole_only or len(needed) == n_subs or not contiguous:
            out.append((coords, ck, 0, chunk_bytes, tuple(c * wi for c, wi in zip(coords, w)),
                        tuple(w), True, chunk_bytes))
            continue
        for sub in sorted(needed):
            rel = tuple(s - c * n for s, c, n in zip(sub, coords, subs_per))
            first = sum(rc * ri * st for rc, ri, st in zip(rel, r, wstrides))
            out.append((coords, ck, first * isz, sub_bytes, tuple(s * ri for s, ri in zip(sub, r)),
                        tuple(r), False, -1))
    return tuple(out)


# -- restore fetch splitting ------------------------------------------------------------------
#
# The reference assembles any target box from whole chunks in host memory, with no size
# ceiling (``chunkstore.py:507-593``).  Here a fetch that does not land contiguously in its
# reader's target goes through device staging, which is bounded.  A fetched box is stored
# row-major and contiguous, so a slab of it along its leading (first non-unit) dimension
# is itself one contiguous byte range of the stored chunk: fetches are cut into such
# slabs — at the target boxes' boundaries first, so each piece can land directly (H2D,
# no kernel, no NVLink hop) in the one target that holds it, then into slabs of at most
# the staging budget.  Every stored byte a target needs is still read exactly once.


def _leading_dim(shape: Sequence[int]) -> int | None:
    for d, e in enumerate(shape):
        if e > 1:
            return d
    return None


def _slab(rel: int, origin: tuple[int, ...], shape: tuple[int, ...], d: int, a: int, b: int,
          row: int) -> tuple[int, int, tuple[int, ...], tuple[int, ...]]:
    """(byte offset, nbytes, origin, shape) of rows [a, b) along dim ``d`` of a box whose
    dims before ``d`` have extent 1 (``row`` = bytes per index of dim ``d``)."""
    o = list(origin)
    s = list(shape)
    o[d] += a
    s[d] = b - a
    return rel + a * row, (b - a) * row, tuple(o), tuple(s)


def cut_rows(rel: int, nbytes: int, origin: tuple[int, ...], shape: tuple[int, ...],
             max_bytes: int) -> list[tuple[int, int, tuple[int, ...], tuple[int, ...]]]:
    """Cut a contiguous box into consecutive contiguous slabs of at most ``max_bytes``
    (descending into the next dimension when one index of the leading one is larger)."""
    if nbytes <= max_bytes:
        return [(rel, nbytes, origin, shape)]
    d = _leading_dim(shape)
    if d is None:  # one element larger than the budget: nothing to cut
        return [(rel, nbytes, origin, shape)]
    row = nbytes // shape[d]
    if row <= max_bytes:
        per = max(1, max_bytes // row)
        return [_slab(rel, origin, shape, d, a, min(a + per, shape[d]), row)
                for a in range(0, shape[d], per)]
    out = []
    for a in range(shape[d]):
        out.extend(cut_rows(*_slab(rel, origin, shape, d, a, a + 1, row), max_bytes))
    return out


def _lands_contiguously(box: tuple[Range, ...], target: tuple[Range, ...]) -> bool:
    if not all(to <= bo and bo + be <= to + te for (bo, be), (to, te) in zip(box, target)):
        return False
    return box_is_contiguous(tuple(e for _, e in target),
                             tuple(bo - to for (bo, _), (to, _) in zip(box, target)),
                             tuple(e for _, e in box))


@functools.lru_cache(maxsize=1 << 12)
def split_geometry(geometry: tuple[tuple, ...], boxes: tuple[tuple[Range, ...], ...],
                   max_bytes: int) -> tuple[tuple, ...]:
    """Refine a restore's fetch geometry (see above): a fetch no target box holds as one
    contiguous run is cut along its leading dimension at the target boxes' boundaries;
    pieces no target needs are dropped; pieces that still land contiguously nowhere are
    cut into slabs of at most ``max_bytes``.  Fetches some target holds contiguously are
    kept whole (they land there directly; replicas are served from the landing copy)."""
    index = BoxIndex(boxes)
    out: list[tuple] = []
    for g in geometry:
        coords, ck, rel, nbytes, origin, shape, whole, obj = g
        box = tuple(zip(origin, shape))
        hits = index.hits(box)
        if any(_lands_contiguously(box, boxes[i]) for i in hits):
            out.append(g)
            continue
        d = _leading_dim(shape)
        pieces = [(rel, nbytes, origin, shape)]
        if d is not None:
            cuts = {0, shape[d]}
            for i in hits:
                o, e = boxes[i][d]
                for c in (o - origin[d], o + e - origin[d]):
                    if 0 < c < shape[d]:
                        cuts.add(c)
            row = nbytes // shape[d]
            cuts_sorted = sorted(cuts)
            pieces = [_slab(rel, origin, shape, d, a, b, row) for a, b in zip(cuts_sorted, cuts_sorted[1:])]
        for prel, pbytes, porigin, pshape in pieces:
            pbox = tuple(zip(porigin, pshape))
            phits = index.hits(pbox)
            if not phits:
                continue  # bytes no target needs are not read
            if any(_lands_contiguously(pbox, boxes[i]) for i in phits):
                out.append((coords, ck, prel, pbytes, porigin, pshape, whole and pbytes == nbytes, obj))
                continue
            for srel, sbytes, sorigin, sshape in cut_rows(prel, pbytes, porigin, pshape, max_bytes):
                if not index.hits(tuple(zip(sorigin, sshape))):
                    continue
                out.append((coords, ck, srel, sbytes, sorigin, sshape, whole and sbytes == nbytes, obj))
    return tuple(out)


def split_fetch(f: Fetch, max_bytes: int) -> list[Fetch]:
    """``f`` as consecutive contiguous slabs of at most ``max_bytes`` (execution-time
    guard for fetches that would need more device staging than the budget)."""
    if f.nbytes <= max_bytes:
        return [f]
    pieces = cut_rows(f.file_off, f.nbytes, f.origin, f.shape, max_bytes)
    if len(pieces) == 1:
        return [f]
    return [Fetch(f.key, "get_range", off, n, o, s, False, f.object_bytes) for off, n, o, s in pieces]


def fetches_at(prefix: str, leaf_path: str, entry: dict, geometry: tuple[tuple, ...]) -> list[Fetch]:
    """Bind a fetch geometry to one leaf's stored chunks (merged-index locations)."""
    locations = entry["chunks"]
    out: list[Fetch] = []
    bound: tuple = ()
    for coords, ck, rel, nbytes, origin, shape, whole_chunk, obj in geometry:
        if not bound or bound[0] != ck:
            loc = locations.get(ck)
            if loc is None:
                raise CorruptionError(f"chunk {ck} of {leaf_path!r} missing from merged index")
            if "f" in loc:
                key = f"{prefix}/process_{loc['p']}/{DATA_DIR}/{loc['f']}"
                bound = (ck, key, int(loc["o"]), "get_range", False)
            else:
                key = f"{prefix}/process_{loc['p']}/" + chunk_object_key(leaf_path, coords)
                bound = (ck, key, 0, "get", True)
        _, key, base, op, whole = bound
        checked = obj if whole else -1  # per-leaf objects: the size a whole read expects
        if whole_chunk:
            out.append(Fetch(key, op, base, nbytes, origin, shape, whole, checked))
        else:
            out.append(Fetch(key, "get_range", base + rel, nbytes, origin, shape, False, checked))
    return out


class ChunkReader:
    """Reads array ranges of a finalized checkpoint through its merged index."""

    def __init__(self, store: Store, ckpt_prefix: str, merged_index: dict, *, gpu: int | None = None,
                 engine_cfg=None):
        self._store = store
        self._prefix = ckpt_prefix.rstrip("/")
        self._arrays = merged_index["arrays"]
        self._gpu = gpu
        self._engine_cfg = engine_cfg

    def metadata_for(self, leaf_path: str) -> ArrayStorageMetadata:
        if leaf_path not in self._arrays:
            raise CorruptionError(f"leaf {leaf_path!r} missing from merged index")
        return ArrayStorageMetadata.from_json(self._arrays[leaf_path])

    def read_range(self, leaf_path: str, ranges: tuple[Range, ...]):
        """The box ``ranges`` of ``leaf_path`` as a fresh CUDA tensor (loading the
        minimal set of read chunks), plus byte stats; ``.cpu()`` it for host bytes."""
        import torch

        from .dtypes import torch_dtype

        meta = self.metadata_for(leaf_path)
        isz = itemsize(meta.dtype)
        ranges = tuple((int(o), int(e)) for o, e in ranges)
        if len(ranges) != meta.rank:
            raise ChunkStoreError(f"rank mismatch reading {leaf_path!r}")
        for (off, ext), g in zip(ranges, meta.global_shape):
            if off < 0 or ext < 0 or off + ext > g:
                raise ChunkStoreError(f"range ({off}, {ext}) outside global extent {g}")
        extents = tuple(e for _, e in ranges)
        gpu = self._gpu if self._gpu is not None else torch.cuda.current_device()
        out = torch.empty(extents, dtype=torch_dtype(meta.dtype), device=torch.device("cuda", gpu))
        # the engine writes `out` on its own streams: the caching allocator may have handed
        # back a block that work queued on the caller's stream still uses
        torch.cuda.current_stream(gpu).synchronize()
        stats = ReadStats(bytes_requested=math.prod(extents) * isz)
        if 0 not in extents:
            fetches = plan_fetches(self._prefix, leaf_path, self._arrays[leaf_path], meta, [ranges])
            dest = Destination(gpu, out.data_ptr(), ranges, isz)
            items = [FetchItem(f, gpu, [dest]) for f in fetches]
            execute_reads(self._store, items, self._engine_cfg)
            stats.bytes_loaded = sum(f.nbytes for f in fetches)
        from . import compat

        if compat.enabled():  # the reference's return type: a host numpy box
            from .treemodel import DenseArray

            return DenseArray(meta.dtype, out).to_numpy(), stats
        return out, stats


# -- restore execution ------------------------------------------------------------------------


@dataclass(slots=True)
class Destination:
    """A target box on a GPU: the tensor at ``address`` holds global box ``ranges``.
    ``src_code``/``dst_code`` (native.DTYPE_CODE) make the copy into it converting (the
    fused load-time cast); ``itemsize`` is then the destination element size."""

    gpu: int
    address: int
    ranges: tuple[Range, ...]
    itemsize: int
    src_code: int = 0
    dst_code: int = 0
    src_itemsize: int = 0


@dataclass(slots=True)
class FetchItem:
    fetch: Fetch
    reader_gpu: int
    consumers: list[Destination] = field(default_factory=list)
    cast_flags: int = 0   # device address of the leaf's check word on the reader GPU


MAX_PIECE_BYTES = 256 << 20


def staging_budget(cfg, concurrent: int = 1) -> int:
    """Largest fetch that may go through device staging: a quarter of the engine's
    staging buffer (several items in flight), at most MAX_PIECE_BYTES."""
    staging = cfg.sizing(concurrent)[2]
    return max(1, min(MAX_PIECE_BYTES, staging // 4))


def _direct_consumer(it: FetchItem) -> tuple[Destination | None, int]:
    """The consumer on the reader GPU the fetched bytes land in as one contiguous run
    without conversion (a direct H2D target), and the landing address."""
    f = it.fetch
    fetched = tuple(zip(f.origin, f.shape))
    for d in it.consumers:
        if d.gpu != it.reader_gpu or d.src_code:
            continue
        if not all(do <= fo and fo + fe <= do + de for (fo, fe), (do, de) in zip(fetched, d.ranges)):
            continue
        dshape = tuple(e for _, e in d.ranges)
        doff = tuple(fo - do for (fo, _), (do, _) in zip(fetched, d.ranges))
        if box_is_contiguous(dshape, doff, f.shape):
            return d, d.address + box_flat_offset(dshape, doff) * d.itemsize
    return None, 0


def _within_staging(items: list[FetchItem], budget: int) -> list[FetchItem]:
    """Items that need device staging (no direct consumer) and exceed ``budget`` become
    several items over consecutive slabs of the fetch (still one read of each byte);
    slabs no consumer meets are not read."""
    out: list[FetchItem] = []
    for it in items:
        if it.fetch.nbytes <= budget or _direct_consumer(it)[0] is not None:
            out.append(it)
            continue
        for f in split_fetch(it.fetch, budget):
            box = tuple(zip(f.origin, f.shape))
            if any(_intersect(box, d.ranges) is not None for d in it.consumers):
                out.append(FetchItem(f, it.reader_gpu, it.consumers, it.cast_flags))
    return out


def execute_reads(store: Store, items: list[FetchItem], engine_cfg=None, concurrent: int = 1,
                  before_engine=None):
    """Fetch every item once onto its reader GPU and scatter it into every consumer
    (local or peer GPUs).  Admission / recording of the get ops as in execute_writes.
    ``before_engine(nbytes)`` runs right before the blocking engine call."""
    from . import native

    if not items:
        return None
    cfg = engine_cfg or native.EngineConfig()
    items = _within_staging(items, staging_budget(cfg, concurrent))
    backend = store.backend
    keys = [it.fetch.key for it in items]
    store.sched_point()
    n_ok, err = backend.admit_bulk("get", keys)
    items = items[:n_ok]
    root = backend.native_root()
    input_index: dict[str, int] = {}
    input_keys: list[str] = []
    for it in items:
        if it.fetch.key not in input_index:
            input_index[it.fetch.key] = len(input_keys)
            input_keys.append(it.fetch.key)
    inputs = np.zeros(len(input_keys), native.INPUT)
    keep_alive = []
    if root is not None:
        paths = native.PathTable([backend.path_of(k) for k in input_keys])
        keep_alive.append(paths)
        inputs["path"] = paths.pointers
        try:
            inputs["size"] = [backend._size(k) for k in input_keys]
        except MissingKeyError:
            raise
    else:
        for i, k in enumerate(input_keys):
            with backend._lock:
                data = backend._get(k)
            arr = np.frombuffer(data, np.uint8)
            keep_alive.append(arr)
            inputs[i]["host"] = arr.ctypes.data if arr.size else 0
            inputs[i]["size"] = arr.size
    for it in items:
        size = int(inputs[input_index[it.fetch.key]]["size"])
        if it.fetch.object_bytes >= 0 and size != it.fetch.object_bytes:  # a per-leaf chunk object
            raise CorruptionError(
                f"chunk object {it.fetch.key!r} has {size} bytes, expected {it.fetch.object_bytes}"
            )
        if it.fetch.file_off + it.fetch.nbytes > size:  # a span of an aggregated data file
            from .errors import BackendError

            raise BackendError(
                f"range [{it.fetch.file_off}, {it.fetch.file_off + it.fetch.nbytes}) outside key "
                f"{it.fetch.key!r} of size {size}"
            )
    ritems = np.zeros(len(items), native.READ_ITEM)
    direct_dst = np.zeros(len(items), np.uint64)
    first_copy = np.zeros(len(items), np.int32)
    n_copies = np.zeros(len(items), np.int32)
    cols: dict[str, list] = {k: [] for k in ("sb", "ss", "so", "db", "ds", "do", "ext", "isz", "sdt", "ddt", "flg")}
    peer_bytes = 0
    for j, it in enumerate(items):
        f = it.fetch
        fetched = tuple(zip(f.origin, f.shape))
        direct, direct_dst[j] = _direct_consumer(it)
        first_copy[j] = len(cols["ext"])
        for d in it.consumers:
            if d is direct:
                continue
            hit = _intersect(fetched, d.ranges)
            if hit is None:
                continue
            cols["sb"].append(0)
            cols["ss"].append(f.shape)
            cols["so"].append(tuple(h - o for (h, _), o in zip(hit, f.origin)))
            cols["db"].append(d.address)
            cols["ds"].append(tuple(e for _, e in d.ranges))
            cols["do"].append(tuple(h - o for (h, _), (o, _) in zip(hit, d.ranges)))
            cols["ext"].append(tuple(e for _, e in hit))
            if d.gpu != it.reader_gpu:  # lands in another GPU's HBM: NVLink (P2P / IPC)
                peer_bytes += math.prod(e for _, e in hit) * d.itemsize
            cols["isz"].append(d.src_itemsize if d.src_code else d.itemsize)
            cols["sdt"].append(d.src_code)
            cols["ddt"].append(d.dst_code)
            cols["flg"].append(it.cast_flags if d.src_code else 0)
        n_copies[j] = len(cols["ext"]) - first_copy[j]
    ritems["input"] = [input_index[it.fetch.key] for it in items]
    ritems["device"] = [it.reader_gpu for it in items]
    ritems["in_off"] = [it.fetch.file_off for it in items]
    ritems["nbytes"] = [it.fetch.nbytes for it in items]
    ritems["direct_dst"] = direct_dst
    ritems["first_copy"] = first_copy
    ritems["n_copies"] = n_copies
    copies = native.copy_table(cols["sb"], cols["ss"], cols["so"], cols["db"], cols["ds"], cols["do"],
                               cols["ext"], cols["isz"], cols["sdt"], cols["ddt"], cols["flg"])
    with native.engine_lease(cfg, concurrent) as eng:
        if before_engine is not None:
            before_engine(int(ritems["nbytes"].sum()))
        stats = eng.load(ritems, inputs, copies)
    native.account_peer(peer_bytes)
    backend.record_bulk(
        store.identity, [it.fetch.op for it in items], [it.fetch.key for it in items],
        [it.fetch.nbytes for it in items], [0] * len(items),
    )
    if err is not None:
        raise err
    return stats


# -- metadata merge ---------------------------------------------------------------------------


def merge_process_indices(store: Store, ckpt_prefix: str, process_count: int) -> dict:
    """Merged index from the per-process documents (``chunkstore.py:603-690``): checks
    that processes agree on every array, no chunk is claimed twice, and every grid is
    complete; payload bytes are never read."""
    prefix = ckpt_prefix.rstrip("/")
    layout: str | None = None
    arrays: dict[str, dict] = {}
    metas: dict[str, ArrayStorageMetadata] = {}
    leaf_sets: list[set[str]] = []
    for p in range(process_count):
        pdir = f"{prefix}/process_{p}"
        try:
            raw = store.get(f"{pdir}/{ARRAY_METADATA_FILE}")
        except MissingKeyError:
            raise ConsistencyError(f"missing array metadata for process {p}") from None
        doc = docio.loads_fast(raw, what=f"process {p} array metadata")
        if layout is None:
            layout = doc.get("layout")
        elif doc.get("layout") != layout:
            raise ConsistencyError(f"process {p} layout {doc.get('layout')!r} != {layout!r}")
        manifest = None
        if layout == AGGREGATED:
            try:
                raw = store.get(f"{pdir}/{MANIFEST_FILE}")
            except MissingKeyError:
                raise ConsistencyError(f"missing manifest for process {p}") from None
            manifest = AggregatedManifest.from_json(docio.loads(raw, what=f"process {p} manifest"))
        entries = doc.get("arrays", {})
        leaf_sets.append(set(entries))
        for leaf, entry in entries.items():
            known = arrays.get(leaf)
            if known is None:
                meta = ArrayStorageMetadata.from_json(entry)
                metas[leaf] = meta
                arrays[leaf] = known = {**meta.to_json(), "sharding": entry.get("sharding"), "chunks": {}}
            elif (entry.get("global_shape") != known["global_shape"] or entry.get("dtype") != known["dtype"]
                  or entry.get("shard_shape") != known["shard_shape"]
                  or entry.get("write_chunk") != known["write_chunk"]
                  or entry.get("read_chunk") != known["read_chunk"] or entry.get("layout") != known["layout"]):
                ArrayStorageMetadata.from_json(entry)  # a malformed entry raises CorruptionError
                raise ConsistencyError(f"process {p} disagrees on storage metadata for {leaf!r}")
            elif known["sharding"] != entry.get("sharding"):
                raise ConsistencyError(f"process {p} disagrees on sharding for {leaf!r}")
            located = known["chunks"]
            for ck in entry.get("chunks", []):
                if ck in located:
                    raise DuplicateChunkError(
                        f"chunk {ck} of {leaf!r} claimed by processes {located[ck]['p']} and {p}"
                    )
                if manifest is not None:
                    fid, off, length = manifest.lookup(f"{leaf}/c.{ck}")
                    located[ck] = {"p": p, "f": fid, "o": off, "l": length}
                else:
                    located[ck] = {"p": p}
    if any(s != set(arrays) for s in leaf_sets):
        raise ConsistencyError("processes disagree on the array leaf set")
    for leaf, entry in arrays.items():
        expected = metas[leaf].total_chunks()
        if len(entry["chunks"]) != expected:
            raise ConsistencyError(f"{leaf!r} has {len(entry['chunks'])} of {expected} chunks")
    return {"format_version": 1, "layout": layout or PER_LEAF, "arrays": arrays}
