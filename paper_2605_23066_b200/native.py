"""ctypes binding of libtvgpu.so (include/tvgpu.h) and the engine pool.

The library is built in-tree by ``paper_2605_23066_b200.build`` (``__graft_entry__.build``)
and loaded from the package directory.  There is no fallback: if the library is missing
or no GPU is visible, every data-path entry point raises ``NativeError``.

Descriptor tables cross the boundary as numpy structured arrays whose layout equals the
C structs (checked against a compiled ``offsetof`` probe in tests/test_native_abi.py), so
a save of thousands of chunks builds its tables with vectorised column writes instead of
one ctypes object per chunk.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path
from typing import Sequence

import numpy as np

from .errors import NativeError

MAX_RANK = 8
LIB_PATH = Path(__file__).resolve().parent / "libtvgpu.so"

TV_OK = 0
TV_ERR_IO = -2  # include/tvgpu.h
POOL_REGISTER = 1  # TV_POOL_REGISTER
POOL_ZERO_COPY = 2  # TV_POOL_ZERO_COPY

# ---- C struct layouts -------------------------------------------------------------------

ARRAY_BOX = np.dtype(
    [("base", "<u8"), ("shape", "<i8", (MAX_RANK,)), ("off", "<i8", (MAX_RANK,))], align=True
)
COPY = np.dtype(
    [("src", ARRAY_BOX), ("dst", ARRAY_BOX), ("ext", "<i8", (MAX_RANK,)), ("rank", "<i4"),
     ("itemsize", "<i4"), ("src_dtype", "<i4"), ("dst_dtype", "<i4"), ("flags", "<u8")],
    align=True,
)

# element type codes of converting copies (include/tvgpu.h TV_DT_*)
DTYPE_CODE = {"f32": 1, "f64": 2, "i32": 3, "i64": 4, "u8": 5, "bool": 6, "bf16": 7}
CAST_OVERFLOW, CAST_NONINTEGRAL, CAST_NONFINITE = 1, 2, 4
WRITE_ITEM = np.dtype(
    [("src", ARRAY_BOX), ("ext", "<i8", (MAX_RANK,)), ("rank", "<i4"), ("itemsize", "<i4"),
     ("file", "<i4"), ("device", "<i4"), ("file_off", "<i8")],
    align=True,
)
OUTPUT = np.dtype([("path", "<u8"), ("host", "<u8"), ("size", "<i8")], align=True)
READ_ITEM = np.dtype(
    [("input", "<i4"), ("device", "<i4"), ("in_off", "<i8"), ("nbytes", "<i8"),
     ("direct_dst", "<u8"), ("first_copy", "<i4"), ("n_copies", "<i4")],
    align=True,
)
INPUT = OUTPUT
STATS = np.dtype(
    [("bytes_device", "<i8"), ("bytes_storage", "<i8"), ("bytes_packed", "<i8"),
     ("kernel_launches", "<i8"), ("dma_copies", "<i8"), ("files", "<i8"),
     ("seconds_total", "<f8"), ("seconds_kernel", "<f8"), ("seconds_io", "<f8"),
     ("seconds_wait_dma", "<f8"), ("seconds_wait_slot", "<f8"), ("recycled_files", "<i8"),
     ("zero_copy_bytes", "<i8"), ("registered_files", "<i8")],
    align=True,
)

# Every symbol include/tvgpu.h declares (tests check the library exports all of them).
EXPORTS = (
    "tv_abi_version", "tv_last_error", "tv_copy_boxes", "tv_copy_bytes", "tv_kernel_timing",
    "tv_kernel_timing_collect", "tv_engine_create",
    "tv_engine_destroy", "tv_engine_save", "tv_engine_load", "tv_enable_peer_access",
    "tv_ipc_export", "tv_ipc_import", "tv_ipc_close", "tv_probe_storage", "tv_probe_pcie",
    "tv_unlink_many", "tv_probe_storage_dma", "tv_engine_save_pooled", "tv_recycle_many",
    "tv_probe_storage_rewrite", "tv_pool_register", "tv_pool_drain", "tv_mapping_stats",
    "tv_mapping_release_all",
)

_lib = None
_lib_lock = threading.Lock()


def _declare(lib: ctypes.CDLL) -> None:
    P, I, L, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "tv_abi_version": (I, []),
        "tv_last_error": (I, [ctypes.c_char_p, ctypes.c_size_t]),
        "tv_copy_boxes": (I, [I, P, I, P]),
        "tv_copy_bytes": (L, [P, I]),
        "tv_kernel_timing": (I, [I]),
        "tv_kernel_timing_collect": (I, [ctypes.POINTER(D), ctypes.POINTER(D), ctypes.POINTER(L),
                                         ctypes.POINTER(L)]),
        "tv_engine_create": (I, [I, L, L, I, ctypes.POINTER(P)]),
        "tv_engine_destroy": (I, [P]),
        "tv_engine_save": (I, [P, P, I, P, I, P]),
        "tv_engine_load": (I, [P, P, I, P, I, P, I, P]),
        "tv_enable_peer_access": (I, [P, I]),
        "tv_ipc_export": (I, [I, ctypes.c_uint64, P, ctypes.POINTER(ctypes.c_uint64)]),
        "tv_ipc_import": (I, [I, P, ctypes.POINTER(ctypes.c_uint64)]),
        "tv_ipc_close": (I, [I, ctypes.c_uint64]),
        "tv_probe_storage": (I, [ctypes.c_char_p, I, L, L, ctypes.POINTER(D), ctypes.POINTER(D)]),
        "tv_probe_pcie": (I, [I, L, I, ctypes.POINTER(D), ctypes.POINTER(D)]),
        "tv_unlink_many": (I, [P, I, I, P]),
        "tv_engine_save_pooled": (I, [P, P, I, P, I, ctypes.c_char_p, I, P]),
        "tv_recycle_many": (I, [P, I, ctypes.c_char_p, I, P]),
        "tv_pool_register": (I, [ctypes.c_char_p, I, ctypes.POINTER(L)]),
        "tv_pool_drain": (I, [ctypes.c_char_p, ctypes.POINTER(L)]),
        "tv_mapping_stats": (I, [ctypes.POINTER(L), ctypes.POINTER(L)]),
        "tv_mapping_release_all": (I, []),
        "tv_probe_storage_rewrite": (I, [ctypes.c_char_p, I, L, L, ctypes.POINTER(D), ctypes.POINTER(D),
                                         ctypes.POINTER(D)]),
        "tv_probe_storage_dma": (I, [ctypes.c_char_p, I, L, L, I, ctypes.POINTER(D), ctypes.POINTER(D),
                                     ctypes.POINTER(D), ctypes.POINTER(D)]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib() -> ctypes.CDLL:
    """The loaded library; raises NativeError when it is absent (no CPU fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise NativeError(
                    f"{LIB_PATH} is missing: build it with `python -m "
                    "paper_2605_23066_b200.build` (there is no CPU fallback)"
                )
            try:
                handle = ctypes.CDLL(str(LIB_PATH))
            except OSError as exc:
                raise NativeError(f"cannot load {LIB_PATH}: {exc}") from exc
            _declare(handle)
            if handle.tv_abi_version() != 2:
                raise NativeError("libtvgpu ABI version mismatch")
            _lib = handle
    return _lib


def last_error() -> str:
    buf = ctypes.create_string_buffer(4096)
    lib().tv_last_error(buf, len(buf))
    return buf.value.decode("utf-8", "replace")


def check(rc: int, what: str) -> None:
    """Raise for a failed call: storage failures (open / pwrite / pread / rename / unlink,
    TV_ERR_IO) as the reference's BackendError — the type its FilesystemBackend raises —
    everything else (CUDA, arguments, memory) as NativeError."""
    if rc != TV_OK:
        msg = f"{what} failed (code {rc}): {last_error()}"
        if rc == TV_ERR_IO:
            from .errors import BackendError

            raise BackendError(msg)
        raise NativeError(msg)


def require_gpu() -> None:
    import torch

    if not torch.cuda.is_available():
        raise NativeError("no CUDA device: the B200 data path has no CPU fallback")


def _ptr(arr: np.ndarray) -> int:
    return arr.ctypes.data if arr.size else 0


# ---- descriptor tables (vectorised column writes) --------------------------------------


def pad_rows(rows: Sequence[Sequence[int]]) -> np.ndarray:
    """(n, MAX_RANK) int64 array of per-dimension values, zero padded."""
    out = np.zeros((len(rows), MAX_RANK), np.int64)
    for i, r in enumerate(rows):
        if r:
            out[i, : len(r)] = r
    return out


def copy_table(src_base, src_shape, src_off, dst_base, dst_shape, dst_off, ext, itemsize,
               src_dtype=None, dst_dtype=None, flags=None) -> np.ndarray:
    """COPY table from per-copy lists (bases ints, shapes/offsets/extents tuples); the
    optional dtype-code / flag-address columns turn rows into converting copies."""
    n = len(ext)
    t = np.zeros(n, COPY)
    if n == 0:
        return t
    t["src"]["base"] = np.asarray(src_base, np.uint64)
    t["src"]["shape"] = pad_rows(src_shape)
    t["src"]["off"] = pad_rows(src_off)
    t["dst"]["base"] = np.asarray(dst_base, np.uint64)
    t["dst"]["shape"] = pad_rows(dst_shape)
    t["dst"]["off"] = pad_rows(dst_off)
    t["ext"] = pad_rows(ext)
    t["rank"] = [len(e) for e in ext]
    t["itemsize"] = itemsize
    if src_dtype is not None:
        t["src_dtype"] = src_dtype
        t["dst_dtype"] = dst_dtype
        t["flags"] = np.asarray(flags, np.uint64)
    return t


def write_table(src_base, src_shape, src_off, ext, itemsize, file, device, file_off) -> np.ndarray:
    n = len(ext)
    t = np.zeros(n, WRITE_ITEM)
    if n == 0:
        return t
    t["src"]["base"] = np.asarray(src_base, np.uint64)
    t["src"]["shape"] = pad_rows(src_shape)
    t["src"]["off"] = pad_rows(src_off)
    t["ext"] = pad_rows(ext)
    t["rank"] = [len(e) for e in ext]
    t["itemsize"] = itemsize
    t["file"] = file
    t["device"] = device
    t["file_off"] = file_off
    return t


# ---- kernels ----------------------------------------------------------------------------


# Process-wide counters of native work (bench.py reports the kernel launches and DMA
# transfers its timed region issued).
_FIELDS = ("kernel_launches", "dma_copies", "bytes_device", "bytes_storage", "bytes_packed", "files",
           "seconds_total", "seconds_io", "seconds_wait_dma", "seconds_wait_slot", "recycled_files",
           "zero_copy_bytes", "registered_files")
TOTALS = {"save": dict.fromkeys(_FIELDS, 0), "load": dict.fromkeys(_FIELDS, 0),
          "kernels": {"kernel_launches": 0}, "peer": {"bytes": 0}}
_totals_lock = threading.Lock()


def _account(kind: str, stats) -> None:
    with _totals_lock:
        for k in _FIELDS:
            TOTALS[kind][k] += stats[k].item()


def account_peer(nbytes: int) -> None:
    """Restore bytes the fan-out kernel stored into another GPU's HBM (NVLink)."""
    with _totals_lock:
        TOTALS["peer"]["bytes"] += int(nbytes)


def totals() -> dict:
    """Combined counters plus the per-kind ("save" / "load") breakdown."""
    with _totals_lock:
        out = {k: TOTALS["save"][k] + TOTALS["load"][k] for k in _FIELDS}
        out["kernel_launches"] += TOTALS["kernels"]["kernel_launches"]
        out["peer_bytes"] = TOTALS["peer"]["bytes"]
        out["save"] = dict(TOTALS["save"])
        out["load"] = dict(TOTALS["load"])
        return out


def copy_boxes(device: int, copies: np.ndarray, stream: int = 0) -> None:
    """One batched box-copy launch on ``device``/``stream`` (COPY-dtype table)."""
    copies = np.ascontiguousarray(copies, dtype=COPY)
    if copies.size == 0:
        return
    check(lib().tv_copy_boxes(device, _ptr(copies), len(copies), stream), "tv_copy_boxes")
    with _totals_lock:
        TOTALS["kernels"]["kernel_launches"] += 1


def kernel_timing(enable: bool) -> None:
    """Bracket every later box-copy / cast launch with CUDA timing events (bench.py)."""
    check(lib().tv_kernel_timing(1 if enable else 0), "tv_kernel_timing")


def kernel_timing_collect() -> dict:
    """Launches recorded since the last collect: summed / longest kernel ms, algorithmic
    HBM bytes (read + write) and count.  Waits for the recorded launches."""
    tot, mx = ctypes.c_double(), ctypes.c_double()
    nbytes, n = ctypes.c_int64(), ctypes.c_int64()
    check(lib().tv_kernel_timing_collect(ctypes.byref(tot), ctypes.byref(mx), ctypes.byref(nbytes),
                                         ctypes.byref(n)), "tv_kernel_timing_collect")
    return {"ms_total": tot.value, "ms_max": mx.value, "bytes": nbytes.value, "launches": n.value}


def enable_peer_access(gpus: Sequence[int]) -> None:
    gpus = sorted(set(int(g) for g in gpus))
    if len(gpus) < 2:
        return
    arr = (ctypes.c_int * len(gpus))(*gpus)
    check(lib().tv_enable_peer_access(arr, len(gpus)), "tv_enable_peer_access")


def ipc_export(device: int, ptr: int) -> tuple[bytes, int]:
    handle = ctypes.create_string_buffer(64)
    off = ctypes.c_uint64()
    check(lib().tv_ipc_export(device, ptr, handle, ctypes.byref(off)), "tv_ipc_export")
    return handle.raw, off.value


def ipc_import(device: int, handle: bytes) -> int:
    out = ctypes.c_uint64()
    buf = ctypes.create_string_buffer(handle, 64)
    check(lib().tv_ipc_import(device, buf, ctypes.byref(out)), "tv_ipc_import")
    return out.value


def ipc_close(device: int, ptr: int) -> None:
    check(lib().tv_ipc_close(device, ptr), "tv_ipc_close")


def unlink_many(paths: Sequence[str], threads: int) -> list[bool]:
    """Remove files on native threads (no interpreter lock held); True = removed, False =
    did not exist.  Raises BackendError on any other failure."""
    if not paths:
        return []
    table = PathTable(list(paths))
    ok = np.zeros(len(paths), np.uint8)
    check(lib().tv_unlink_many(table.pointers.ctypes.data, len(paths), int(threads), ok.ctypes.data),
          "tv_unlink_many")
    return [bool(x) for x in ok]


def recycle_many(paths: Sequence[str], pool_dir: str, threads: int) -> list[bool]:
    """Retire files into the recycle pool ``pool_dir`` (``<pool_dir>/<size>/<name>``,
    renamed on native threads; unrenameable files are unlinked).  True = retired, False =
    did not exist.  Raises BackendError on any other failure."""
    if not paths:
        return []
    table = PathTable(list(paths))
    ok = np.zeros(len(paths), np.uint8)
    check(lib().tv_recycle_many(table.pointers.ctypes.data, len(paths), pool_dir.encode(), int(threads),
                                ok.ctypes.data), "tv_recycle_many")
    return [bool(x) for x in ok]


def pool_register(pool_dir: str, threads: int = 4) -> int:
    """Map + register (CUDA) every not-yet-registered recycle-pool file on a RAM-backed
    filesystem; bytes registered now (0 without a GPU)."""
    n = ctypes.c_int64()
    check(lib().tv_pool_register(pool_dir.encode(), int(threads), ctypes.byref(n)), "tv_pool_register")
    return n.value


def pool_drain(pool_dir: str) -> int:
    """Release the registrations of, and unlink, every pool file; bytes freed."""
    n = ctypes.c_int64()
    check(lib().tv_pool_drain(pool_dir.encode(), ctypes.byref(n)), "tv_pool_drain")
    return n.value


def mapping_stats() -> tuple[int, int]:
    files, nbytes = ctypes.c_int64(), ctypes.c_int64()
    check(lib().tv_mapping_stats(ctypes.byref(files), ctypes.byref(nbytes)), "tv_mapping_stats")
    return files.value, nbytes.value


class SavePathChooser:
    """Per-GPU choice between the two ways a save can move bytes into recycled files:
    zero-copy (D2H straight into the registered page-cache pages) or the pinned slot ring
    + pwrite.  Which is faster depends on the box: one GPU alone streams 54 GB/s
    zero-copy vs 40 through the slots, while on some 4-GPU boxes three GPUs sharing a
    host-side DMA path get only ~21 GB/s each zero-copy
    (profiles/r02_bench_c2_n4_allzc.json vs r02_bench_c2_n4_4gpu_box.json).

    Keys are (GPU, save-size bucket): rates of a 4 GB and an 80 GB save are not
    comparable.  A bucket with both rates uses the faster path; a bucket without them
    follows its GPU's overall verdict when the GPU has one (no exploration on the
    critical path of, e.g., a Checkpointer loop that starts after a warm-up); otherwise
    each path is tried once (a zero-copy save that had to register new files is a
    warm-up and not scored).  A close call (< 25 % apart) is re-tried every ``RETRY``
    saves."""

    RETRY = 64
    CLOSE = 1.25

    def __init__(self):
        self._lock = threading.Lock()
        self._state: dict = {}

    def _entry(self, key) -> dict:
        return self._state.setdefault(key, {"rate": {True: None, False: None}, "n": 0})

    def choose(self, key) -> bool:
        """True = zero-copy for this save."""
        env = os.environ.get("TVGPU_SAVE_PATH", "auto")
        if env in ("zero_copy", "slots"):
            return env == "zero_copy"
        gpu = key[0] if isinstance(key, tuple) else key
        with self._lock:
            st = self._entry(key)
            st["n"] += 1
            rz, rs = st["rate"][True], st["rate"][False]
            if rz is not None and rs is not None:
                best = rz >= rs
                close = max(rz, rs) < self.CLOSE * min(rz, rs)
                return (not best) if close and st["n"] % self.RETRY == 0 else best
            g = self._state.get(("gpu", gpu))
            if g is not None and g["rate"][True] is not None and g["rate"][False] is not None:
                return g["rate"][True] >= g["rate"][False]
            return rz is None

    def record(self, key, zero_copy: bool, nbytes: int, seconds: float, warm_up: bool) -> None:
        """Score a save.  Warm-ups (files registered) are not scored, and neither is the
        first zero-copy save after one: the first DMA into freshly registered pages runs
        at a fraction of the link rate (the I/O mappings are populated on first touch)."""
        if seconds <= 0 or nbytes <= 0:
            return
        gpu = key[0] if isinstance(key, tuple) else key
        rate = nbytes / seconds
        with self._lock:
            st = self._entry(key)
            if warm_up:
                st["skip_zc"] = 1
                return
            if zero_copy and st.get("skip_zc", 1) > 0:
                st["skip_zc"] = st.get("skip_zc", 1) - 1
                return
            for k in (key, ("gpu", gpu)):
                st = self._entry(k)
                old = st["rate"][zero_copy]
                st["rate"][zero_copy] = rate if old is None else 0.5 * old + 0.5 * rate

    def snapshot(self) -> dict:
        with self._lock:
            return {str(k): {"zero_copy_GBps": None if v["rate"][True] is None else round(v["rate"][True] / 1e9, 2),
                             "slots_GBps": None if v["rate"][False] is None else round(v["rate"][False] / 1e9, 2)}
                    for k, v in self._state.items()}


SAVE_PATHS = SavePathChooser()


def probe_storage(directory: str, threads: int, file_bytes: int, block_bytes: int) -> tuple[float, float]:
    w, r = ctypes.c_double(), ctypes.c_double()
    check(
        lib().tv_probe_storage(directory.encode(), threads, file_bytes, block_bytes,
                               ctypes.byref(w), ctypes.byref(r)),
        "tv_probe_storage",
    )
    return w.value, r.value


def probe_storage_rewrite(directory: str, threads: int, file_bytes: int,
                          block_bytes: int) -> tuple[float, float, float]:
    """(fresh write, rewrite in place, read) GB/s on the same files."""
    w, rw, r = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    check(lib().tv_probe_storage_rewrite(directory.encode(), threads, file_bytes, block_bytes,
                                         ctypes.byref(w), ctypes.byref(rw), ctypes.byref(r)),
          "tv_probe_storage_rewrite")
    return w.value, rw.value, r.value


def probe_storage_dma(directory: str, threads: int, file_bytes: int, block_bytes: int,
                      device: int) -> tuple[float, float, float, float]:
    """(write, read, D2H, H2D) GB/s with the storage probe and a DMA loop running at once."""
    os.makedirs(directory, exist_ok=True)
    w, r, d2h, h2d = (ctypes.c_double() for _ in range(4))
    check(lib().tv_probe_storage_dma(directory.encode(), threads, file_bytes, block_bytes, device,
                                     ctypes.byref(w), ctypes.byref(r), ctypes.byref(d2h),
                                     ctypes.byref(h2d)), "tv_probe_storage_dma")
    return w.value, r.value, d2h.value, h2d.value


def probe_pcie(device: int, nbytes: int = 1 << 30, reps: int = 3) -> tuple[float, float]:
    d2h, h2d = ctypes.c_double(), ctypes.c_double()
    check(lib().tv_probe_pcie(device, nbytes, reps, ctypes.byref(d2h), ctypes.byref(h2d)),
          "tv_probe_pcie")
    return d2h.value, h2d.value


# ---- engine --------------------------------------------------------------------------------


class PathTable:
    """NUL-terminated path strings kept alive for one engine call."""

    def __init__(self, paths: Sequence[str | None]):
        encoded = [(p.encode() + b"\0") if p else b"" for p in paths]
        self._blob = ctypes.create_string_buffer(b"".join(encoded) or b"\0")
        base = ctypes.addressof(self._blob)
        offs = np.zeros(len(encoded), np.uint64)
        pos = 0
        for i, e in enumerate(encoded):
            offs[i] = (base + pos) if e else 0
            pos += len(e)
        self.pointers = offs


class Engine:
    """One libtvgpu engine: pinned slot ring + storage threads (+ per-device staging)."""

    def __init__(self, n_slots: int, slot_bytes: int, staging_bytes: int, threads: int):
        self.config = (n_slots, slot_bytes, staging_bytes, threads)
        self.cpus: set[int] | None = None  # NUMA placement of its threads (_create_engine)
        handle = ctypes.c_void_p()
        check(lib().tv_engine_create(n_slots, slot_bytes, staging_bytes, threads,
                                     ctypes.byref(handle)), "tv_engine_create")
        self._h = handle

    def close(self) -> None:
        if self._h:
            lib().tv_engine_destroy(self._h)
            self._h = None

    def save(self, items: np.ndarray, outputs: np.ndarray, pool_dir: str | None = None,
             register: bool = False, zero_copy: bool = False) -> np.ndarray:
        """Write every item into its output; with ``pool_dir`` outputs reuse recycled
        files of their exact size; ``register`` registers first-claimed ones with CUDA,
        ``zero_copy`` DMAs straight into registered ones (see tv_engine_save_pooled)."""
        stats = np.zeros(1, STATS)
        items = np.ascontiguousarray(items, WRITE_ITEM)
        outputs = np.ascontiguousarray(outputs, OUTPUT)
        flags = (POOL_REGISTER if register else 0) | (POOL_ZERO_COPY if zero_copy else 0)
        with _bound_to(self.cpus):
            rc = lib().tv_engine_save_pooled(self._h, _ptr(items), len(items), _ptr(outputs), len(outputs),
                                             pool_dir.encode() if pool_dir else None, flags,
                                             stats.ctypes.data)
        _account("save", stats[0])
        check(rc, "tv_engine_save")
        return stats[0]

    def load(self, items: np.ndarray, inputs: np.ndarray, copies: np.ndarray) -> np.ndarray:
        stats = np.zeros(1, STATS)
        items = np.ascontiguousarray(items, READ_ITEM)
        inputs = np.ascontiguousarray(inputs, INPUT)
        copies = np.ascontiguousarray(copies, COPY)
        with _bound_to(self.cpus):
            rc = lib().tv_engine_load(self._h, _ptr(items), len(items), _ptr(inputs), len(inputs),
                                      _ptr(copies), len(copies), stats.ctypes.data)
        _account("load", stats[0])
        check(rc, "tv_engine_load")
        return stats[0]


def _llc_bytes() -> int:
    """Total last-level cache of the host (sum over distinct L3 instances), 0 if unknown."""
    import glob

    seen, total = set(), 0
    for path in glob.glob("/sys/devices/system/cpu/cpu*/cache/index3"):
        try:
            with open(f"{path}/shared_cpu_list") as f:
                key = f.read().strip()
            if key in seen:
                continue
            seen.add(key)
            with open(f"{path}/size") as f:
                txt = f.read().strip().upper()
            mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}.get(txt[-1], 1)
            total += int(txt.rstrip("KMG")) * mult
        except OSError:
            continue
    return total


def _host_cores() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 8)


class EngineConfig:
    """Pipeline sizing.

    threads  — host cores shared by the engines running at once on this box (the
               threads runtime's processes, or torchrun's LOCAL_WORLD_SIZE ranks), minus
               one core per engine for its producer when an engine has >= 8 cores;
    n_slots  — 2 pinned slots per storage thread (fewer starves the readers);
    slot     — 4 MiB for a single engine (fewer, larger DMAs); with several engines
               2 MiB, or 1 MiB when the rings of all engines would not fit the host's
               last-level cache (the DMA'd bytes are re-read by pwrite / the H2D from the
               LLC).  Measured best on these boxes (profiles/r01_engine_sweep_*.jsonl,
               r01_ab_slot_*.txt: at 4 engines 1 MiB > 2 MiB > 4 MiB).
    """

    def __init__(self, slot_bytes: int | None = None, n_slots: int | None = None,
                 staging_bytes: int | None = None, threads: int | None = None):
        env = os.environ
        self._slot_bytes = slot_bytes or (int(env["TVGPU_SLOT_BYTES"]) if "TVGPU_SLOT_BYTES" in env else None)
        self._n_slots = n_slots or (int(env["TVGPU_SLOTS"]) if "TVGPU_SLOTS" in env else None)
        self._staging = staging_bytes or (int(env["TVGPU_STAGING_BYTES"]) if "TVGPU_STAGING_BYTES" in env else None)
        self.threads = threads or (int(env["TVGPU_THREADS"]) if "TVGPU_THREADS" in env else None)

    def _engines(self, concurrent: int) -> int:
        return max(concurrent, int(os.environ.get("LOCAL_WORLD_SIZE", "1")))

    def threads_for(self, concurrent: int) -> int:
        """Storage threads per engine: the host's cores minus one per engine (its producer
        thread and the CUDA driver need a core; measured better than all cores)."""
        if self.threads:
            return self.threads
        engines = self._engines(concurrent)
        per = _host_cores() // engines
        # a core for the producer only when there are >= 8 per engine (measured: 15 of 16
        # and 7 of 8 beat all cores; 4 of 4 beats 3 — profiles/r01_ab_threads_*.txt)
        return max(2, min(64, per - 1 if per >= 8 else per))

    def sizing(self, concurrent: int) -> tuple[int, int, int, int]:
        """(n_slots, slot_bytes, staging_bytes, threads) for an engine of this box."""
        threads = self.threads_for(concurrent)
        n_slots = self._n_slots or max(16, 2 * threads)
        slot = self._slot_bytes
        if slot is None:
            engines = self._engines(concurrent)
            if engines == 1:
                # one engine owns the host: fewer, larger DMAs (measured +9 % restore on a
                # huge-page tmpfs, neutral on /dev/shm: profiles/r01_ab_slot_2m_vs_4m_*.txt)
                slot = 4 << 20
            else:
                llc = _llc_bytes()
                ring_all = (2 << 20) * n_slots * engines
                slot = (2 << 20) if (llc == 0 or ring_all <= 1.25 * llc) else (1 << 20)
        staging = self._staging or max(n_slots * slot, 1 << 30)
        return n_slots, slot, staging, threads


def parse_cpulist(text: str) -> set[int]:
    """Linux cpulist syntax ("0-3,8,10-11") -> CPU ids."""
    out: set[int] = set()
    for part in text.strip().split(","):
        if not part:
            continue
        lo, _, hi = part.partition("-")
        out.update(range(int(lo), int(hi or lo) + 1))
    return out


def numa_local_cpus(pci_address: str, sysfs: str = "/sys", force: bool = False) -> set[int] | None:
    """CPUs of the NUMA node a PCI device (the GPU) hangs off, when the host has more than
    one node with CPUs — else None (one node: nothing to place; ``force`` places anyway,
    for testing the path on single-node boxes)."""
    import glob

    nodes = 0
    for node in glob.glob(f"{sysfs}/devices/system/node/node[0-9]*"):
        try:
            with open(f"{node}/cpulist") as f:
                nodes += bool(parse_cpulist(f.read()))
        except OSError:
            continue
    if nodes < 2 and not force:
        return None
    try:
        with open(f"{sysfs}/bus/pci/devices/{pci_address}/local_cpulist") as f:
            cpus = parse_cpulist(f.read())
    except (OSError, ValueError):
        return None
    return cpus or None


_placement: dict = {}


def _engine_cpus() -> set[int] | None:
    """Where a new engine's storage threads and pinned ring go: the CPUs local to this
    rank's GPU under torchrun (one GPU per rank, LOCAL_WORLD_SIZE > 1) on multi-node
    hosts, intersected with the process's allowed CPUs.  TVGPU_NUMA=0 disables,
    TVGPU_NUMA=force applies it on single-node hosts too."""
    mode = os.environ.get("TVGPU_NUMA", "auto")
    if mode == "0" or not hasattr(os, "sched_setaffinity"):
        return None
    if mode != "force" and int(os.environ.get("LOCAL_WORLD_SIZE", "1")) <= 1:
        return None
    import torch

    def local_of(gpu: int) -> set[int] | None:
        prop = torch.cuda.get_device_properties(gpu)
        addr = f"{prop.pci_domain_id:04x}:{prop.pci_bus_id:02x}:{prop.pci_device_id:02x}.0"
        return numa_local_cpus(addr, force=mode == "force")

    gpu = torch.cuda.current_device()
    local = local_of(gpu)
    if local is None:
        return None
    allowed = os.sched_getaffinity(0)
    cpus = local & allowed
    # Bind only when this node's share of the local ranks' GPUs does not exceed its share
    # of the CPUs (the per-engine thread count assumes an even split of the host's cores).
    ranks = min(int(os.environ.get("LOCAL_WORLD_SIZE", "1")), torch.cuda.device_count())
    same = sum(1 for g in range(ranks) if local_of(g) == local) or 1
    if not cpus or same * len(allowed) > len(cpus) * max(ranks, 1) * 1.01:
        return None
    _placement.update({"gpu": gpu, "cpus": len(cpus), "ranks_on_node": same})
    return cpus


def placement() -> dict:
    """The NUMA placement applied to this process's engines ({} when none)."""
    return dict(_placement)


class _bound_to:
    """Run the calling thread on ``cpus`` for the duration (no-op for None).  Threads it
    starts inherit the mask (the engine's storage threads are started per operation)."""

    def __init__(self, cpus: set[int] | None):
        self.cpus, self.before = cpus, None

    def __enter__(self):
        if self.cpus is not None:
            self.before = os.sched_getaffinity(0)
            os.sched_setaffinity(0, self.cpus)

    def __exit__(self, *exc):
        if self.before is not None:
            os.sched_setaffinity(0, self.before)
            self.before = None


def _create_engine(key: tuple) -> Engine:
    """Create an engine bound to the GPU's local CPUs (when placed): its pinned ring is
    allocated, and its storage threads run and fill the page cache, on the GPU's node."""
    cpus = _engine_cpus()
    with _bound_to(cpus):
        engine = Engine(*key)
    engine.cpus = cpus
    return engine


_pool: dict[tuple, list[Engine]] = {}
_pool_lock = threading.Lock()


class engine_lease:
    """Context manager borrowing an idle engine of the given sizing from the pool."""

    def __init__(self, cfg: EngineConfig, concurrent: int):
        self.key = cfg.sizing(concurrent)
        self.engine: Engine | None = None

    def __enter__(self) -> Engine:
        require_gpu()
        with _pool_lock:
            idle = _pool.setdefault(self.key, [])
            self.engine = idle.pop() if idle else None
        if self.engine is None:
            self.engine = _create_engine(self.key)
        return self.engine

    def __exit__(self, *exc) -> None:
        with _pool_lock:
            _pool.setdefault(self.key, []).append(self.engine)


def release_pool() -> None:
    """Destroy every pooled engine (frees pinned memory)."""
    with _pool_lock:
        for engines in _pool.values():
            for e in engines:
                e.close()
        _pool.clear()
