"""ORACLE — test infrastructure only, never product code.

A CPU restatement (numpy, single thread) of the reference's save/restore data path
(treevault, /root/reference/pkg/src/treevault): given global host arrays, shardings and
save options it produces every file of the checkpoint — chunk payloads, aggregated data
files, manifests, per-process metadata, merged index, global metadata, documents and the
commit marker — and, for a restore, the bytes each target shard must hold plus the
per-process payload bytes the reference reads.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import this module.  It is pinned against the reference's own outputs: the golden
fixtures in tests/golden/*.json were produced by running the real reference
(tests/golden/gen_golden.py) and tests/test_oracle_golden.py checks this restatement
reproduces every stored byte (sha256) and every read counter of them.

Inputs use the neutral notation of tests/golden/cases.py.
"""

from __future__ import annotations

import itertools
import json
import math
import os
from typing import Any

import numpy as np

ITEMSIZE = {"f32": 4, "f64": 8, "i32": 4, "i64": 8, "u8": 1, "bool": 1, "bf16": 2}


def canonical(obj: Any) -> bytes:
    """docio.py:16-19 — sorted keys, compact separators, UTF-8."""
    return json.dumps(obj, sort_keys=True, separators=(",", ":"), ensure_ascii=False).encode("utf-8")


# -- sharding (sharding.py:55-282) ------------------------------------------------------------


class Mesh:
    def __init__(self, axes, process_count, replica_axis=None):
        self.names = [n for n, _ in axes]
        self.sizes = [int(s) for _, s in axes]
        n = math.prod(self.sizes)
        per = n // process_count
        self.devices = list(range(n))                       # sharding.py:71-77
        self.proc = [d // per for d in self.devices]
        self.replica_axis = replica_axis

    def coords(self, pos):
        return tuple(int(c) for c in np.unravel_index(pos, self.sizes)) if self.sizes else ()

    def describe(self):
        return {"axes": [[n, s] for n, s in zip(self.names, self.sizes)],
                "devices": self.devices, "device_processes": self.proc}


class Spec:
    def __init__(self, mesh: Mesh, entries, shape):
        self.mesh, self.entries, self.shape = mesh, tuple(entries), tuple(shape)

    def shard_shape(self):
        return tuple(g if a is None else g // self.mesh.sizes[self.mesh.names.index(a)]
                     for g, a in zip(self.shape, self.entries))

    def replication(self):                                  # sharding.py:171-177
        used = {a for a in self.entries if a is not None}
        return math.prod(s for n, s in zip(self.mesh.names, self.mesh.sizes) if n not in used)

    def shards(self):
        """[(device, ranges, replica_ordinal)] in mesh order (sharding.py:201-231)."""
        m, ss = self.mesh, self.shard_shape()
        used = {m.names.index(a) for a in self.entries if a is not None}
        free = [i for i in range(len(m.names)) if i not in used]
        out = []
        for pos, dev in enumerate(m.devices):
            c = m.coords(pos)
            ranges = tuple((0, g) if a is None else (c[m.names.index(a)] * s, s)
                           for g, s, a in zip(self.shape, ss, self.entries))
            ordinal = int(np.ravel_multi_index([c[i] for i in free], [m.sizes[i] for i in free])) if free else 0
            out.append((dev, ranges, ordinal))
        return out

    def describe(self):
        d = self.mesh.describe()
        d["spec"] = list(self.entries)
        d["global_shape"] = list(self.shape)
        return d


def largest_dim(ext):
    return int(np.argmax(np.asarray(ext))) if len(ext) else None  # first max = lowest index


def replica_segment(ranges, n, ordinal):
    """sharding.py:258-282 — ceil split of the largest dim."""
    if n == 1:
        return ranges
    ext = [e for _, e in ranges]
    ax = largest_dim(ext)
    off, e = ranges[ax]
    if e == 0:
        return ranges if ordinal == 0 else None
    seg = -(-e // n)
    lo, hi = min(ordinal * seg, e), min(ordinal * seg + seg, e)
    if lo == hi:
        return None
    r = list(ranges)
    r[ax] = (off + lo, hi - lo)
    return tuple(r)


def write_ranges(spec: Spec | None, shape, p, replica_parallel):
    """save_pipeline.py:141-168."""
    if spec is None:
        return [tuple((0, e) for e in shape)] if p == 0 else []
    if replica_parallel and spec.replication() > 1:
        n = spec.replication()
        out = []
        for dev, ranges, ordinal in spec.shards():
            if spec.mesh.proc[dev] == p:
                seg = replica_segment(ranges, n, ordinal)
                if seg is not None:
                    out.append(seg)
        return out
    return [r for d, r, o in spec.shards() if o == 0 and spec.mesh.proc[d] == p]


# -- chunk grid (chunkstore.py:145-246) ----------------------------------------------------------


def write_chunk_of(shard, n_segments):
    if n_segments <= 1 or not shard or 0 in shard:
        return tuple(shard)
    ax = largest_dim(shard)
    out = list(shard)
    out[ax] = math.gcd(-(-shard[ax] // n_segments), shard[ax])
    return tuple(out)


def read_chunk_of(write, dtype, target):
    if target is None:
        return tuple(write)
    isz = ITEMSIZE[dtype]
    c = list(write)
    if 0 in c:
        return tuple(c)
    for d in sorted(range(len(c)), key=lambda i: (-write[i], i)):
        while c[d] > 1 and math.prod(c) * isz > target:
            if c[d] % 2 == 0:
                c[d] //= 2
            else:
                f = next(k for k in range(3, c[d] + 1, 2) if c[d] % k == 0)
                c[d] //= f
    return tuple(c)


def cells(ranges, steps):
    if any(e == 0 for _, e in ranges):
        return []
    return list(itertools.product(*[range(o // s, (o + e - 1) // s + 1) for (o, e), s in zip(ranges, steps)]))


def ckey(coords):
    return ".".join(str(c) for c in coords) if coords else "0"


# -- trees (treemodel.py:193-290, 506-516) -----------------------------------------------------


def is_leaf(node):
    return isinstance(node, tuple) and bool(node) and node[0] in ("array", "scalar", "text")


def flat(node, prefix=""):
    if is_leaf(node):
        return [(prefix, node)]
    out = []
    items = sorted(node.items()) if isinstance(node, dict) else [(str(i), c) for i, c in enumerate(node)]
    for k, child in items:
        out.extend(flat(child, f"{prefix}/{k}" if prefix else k))
    return out


def skeleton(node):
    if is_leaf(node):
        if node[0] == "array":
            leaf = {"variant": "array", "dtype": node[1], "shape": list(node[2].shape)}
        elif node[0] == "scalar":
            leaf = {"variant": "scalar", "dtype": node[1]}
        else:
            leaf = {"variant": "text"}
        return {"kind": "leaf", "leaf": leaf}
    if isinstance(node, dict):
        return {"kind": "dict", "children": {k: skeleton(v) for k, v in node.items()}}
    return {"kind": "tuple" if isinstance(node, tuple) else "list", "children": [skeleton(v) for v in node]}


def scalar_value(dtype, value):
    if dtype == "bool":
        return bool(value)
    if dtype in ("f32", "f64"):
        v = float(np.dtype("<f4" if dtype == "f32" else "<f8").type(value))
        return v if math.isfinite(v) else repr(v)
    return int(value)


def inline_doc(leaf):
    if leaf[0] == "scalar":
        return {"variant": "scalar", "dtype": leaf[1], "value": scalar_value(leaf[1], leaf[2])}
    return {"variant": "text", "value": leaf[1]}


# -- save ------------------------------------------------------------------------------------------


def expected_checkpoint(tree: dict, shard_specs: dict, options: dict, process_count: int,
                        backend: str, path: str = "ckpt/run") -> dict[str, bytes]:
    """Every key → bytes of the finalized checkpoint (reference semantics)."""
    layout = options.get("layout", "per_leaf")
    sub_target = options.get("subchunk_target_bytes")
    rp = options.get("replica_parallel", False)
    target = options.get("target_file_bytes", 64 * 1024 * 1024)
    commit = "indicator" if backend == "mem" else "rename"
    files: dict[str, bytes] = {}
    descriptors, trees, inline, docs = [], {}, {}, {}
    arrays = {}   # scoped -> (leaf, spec or None)
    for name in sorted(tree):
        value = tree[name]
        if isinstance(value, tuple) and value and value[0] == "json":
            descriptors.append((name, "json"))
            docs[name] = value[1]
            continue
        if isinstance(value, tuple) and value and value[0] == "stateful":
            descriptors.append((name, "stateful"))
            docs[name] = {"index": value[1]}
            continue
        descriptors.append((name, "tree"))
        trees[name] = skeleton(value)
        inl = {}
        for p, leaf in flat(value):
            if leaf[0] == "array":
                raw = shard_specs.get(name, {}).get(p)
                spec = None
                if raw is not None:
                    axes, P, ra, entries = raw
                    spec = Spec(Mesh(axes, P, ra), entries, leaf[2].shape)
                arrays[f"{name}/{p}" if p else name] = (leaf, spec)
            else:
                inl[p] = inline_doc(leaf)
        if inl:
            inline[name] = inl
    gdoc = {
        "format_version": 1,
        "checkpointables": [{"name": n, "handler": h} for n, h in sorted(descriptors)],
        "trees": trees, "inline": inline, "layout": layout, "commit_style": commit,
    }
    files[f"{path}/global_metadata.json"] = canonical(gdoc)
    for name, doc in docs.items():
        files[f"{path}/{name}/data.json"] = canonical(doc)
    metas = {}
    for scoped, (leaf, spec) in arrays.items():
        shape = leaf[2].shape
        shard = spec.shard_shape() if spec else tuple(shape)
        w = write_chunk_of(shard, spec.replication() if (spec and rp) else 1)
        metas[scoped] = {
            "global_shape": list(shape), "dtype": leaf[1], "shard_shape": list(shard),
            "write_chunk": list(w), "read_chunk": list(read_chunk_of(w, leaf[1], sub_target)),
            "layout": layout,
        }
    merged = {}
    for p in range(process_count):
        pdir = f"{path}/process_{p}"
        buf, fid, manifest = bytearray(), 0, {}
        adoc = {}
        for scoped in sorted(arrays):
            leaf, spec = arrays[scoped]
            data = leaf[2]
            w = tuple(metas[scoped]["write_chunk"])
            chunks = []
            for ranges in write_ranges(spec, data.shape, p, rp):
                for coords in cells(ranges, w):
                    sel = tuple(slice(c * s, (c + 1) * s) for c, s in zip(coords, w))
                    payload = np.ascontiguousarray(data[sel]).tobytes()     # chunkstore.py:392
                    chunks.append(ckey(coords))
                    rel = f"{scoped}/c.{ckey(coords)}"
                    if layout == "per_leaf":
                        files[f"{pdir}/{rel}"] = payload
                    else:                                                   # chunkstore.py:409-417
                        if buf and len(buf) + len(payload) > target:
                            files[f"{pdir}/d/{fid}"] = bytes(buf)
                            buf, fid = bytearray(), fid + 1
                        manifest[rel] = [fid, len(buf), len(payload)]
                        buf.extend(payload)
            adoc[scoped] = {**metas[scoped], "sharding": spec.describe() if spec else None,
                            "chunks": sorted(chunks)}
            entry = merged.setdefault(scoped, {**metas[scoped], "sharding": adoc[scoped]["sharding"], "chunks": {}})
            for ck in chunks:
                loc = {"p": p}
                if layout == "aggregated":
                    f, o, l = manifest[f"{scoped}/c.{ck}"]
                    loc.update({"f": f, "o": o, "l": l})
                entry["chunks"][ck] = loc
        if layout == "aggregated":
            if buf:
                files[f"{pdir}/d/{fid}"] = bytes(buf)
            files[f"{pdir}/manifest.json"] = canonical(
                {"target_file_bytes": target, "entries": dict(sorted(manifest.items()))})
        files[f"{pdir}/array_metadata.json"] = canonical(
            {"format_version": 1, "layout": layout, "arrays": adoc})
    files[f"{path}/merged_index.json"] = canonical({"format_version": 1, "layout": layout, "arrays": merged})
    if commit == "indicator":
        files[f"{path}/COMMIT"] = b"COMMIT\n"
    return files


# -- restore -----------------------------------------------------------------------------------


def fetch_bytes(meta: dict, requests) -> int:
    """Payload bytes the reference loads for a set of range requests of ONE process
    (chunkstore.py:537-578: whole chunk if every subchunk is needed or subchunks are not
    contiguous, else one span per needed subchunk), summed per request."""
    w, r = tuple(meta["write_chunk"]), tuple(meta["read_chunk"])
    isz = ITEMSIZE[meta["dtype"]]
    partial = [d for d in range(len(w)) if r[d] != w[d]]
    contiguous = not partial or all(r[d] == 1 for d in range(partial[-1]))
    n_sub = math.prod(wi // ri for wi, ri in zip(w, r))
    total = 0
    for ranges in requests:
        for coords in cells(ranges, w):
            cell = tuple((c * s, s) for c, s in zip(coords, w))
            hit = tuple((max(a, b), min(a + e, b + f) - max(a, b)) for (a, e), (b, f) in zip(ranges, cell))
            needed = len(cells(hit, r))
            total += (math.prod(w) if needed == n_sub or not contiguous else needed * math.prod(r)) * isz
    return total


def reference_read_bytes(tree: dict, metas_by_scoped: dict, target_specs: dict, process_count: int,
                         broadcast: bool) -> dict[int, int]:
    """Per-process chunk payload bytes of the reference's load (load_pipeline.py:406-442):
    each process reads its devices' target ranges, deduplicated within the process;
    broadcast restricts readers to replica group 0; unsharded targets read on process 0."""
    out = {p: 0 for p in range(process_count)}
    for scoped, meta in metas_by_scoped.items():
        spec = target_specs.get(scoped)
        if spec is None:
            out[0] += fetch_bytes(meta, [tuple((0, g) for g in meta["global_shape"])])
            continue
        mesh = spec.mesh
        allowed = None
        if broadcast:
            ax = mesh.names.index(mesh.replica_axis)
            allowed = {d for pos, d in enumerate(mesh.devices) if mesh.coords(pos)[ax] == 0}
        for p in range(process_count):
            seen = []
            for dev, ranges, _ in spec.shards():
                if mesh.proc[dev] != p or (allowed is not None and dev not in allowed):
                    continue
                if ranges not in seen:
                    seen.append(ranges)
            out[p] += fetch_bytes(meta, seen)
    return out


def expected_shards(global_array: np.ndarray, spec: Spec | None) -> dict[int, bytes]:
    """Bytes each target device must hold after a restore (global[ranges])."""
    if spec is None:
        return {-1: np.ascontiguousarray(global_array).tobytes()}
    return {dev: np.ascontiguousarray(global_array[tuple(slice(o, o + e) for o, e in ranges)]).tobytes()
            for dev, ranges, _ in spec.shards()}


# -- CPU baseline: the port writing / reading a real directory -------------------------------------


def save_to_directory(root: str, files: dict[str, bytes]) -> int:
    """FilesystemBackend._put semantics (backend.py:398-403): <file>.partial + rename."""
    total = 0
    for key, data in files.items():
        dst = os.path.join(root, *key.split("/"))
        os.makedirs(os.path.dirname(dst), exist_ok=True)
        with open(dst + ".partial", "wb") as f:
            f.write(data)
        os.replace(dst + ".partial", dst)
        total += len(data)
    return total


def _read_range(root: str, path: str, scoped: str, entry: dict, ranges) -> np.ndarray:
    """chunkstore.py:507-593 for whole-chunk fetches of per-leaf files."""
    w = tuple(entry["write_chunk"])
    dt = {"f32": "<f4", "f64": "<f8", "i32": "<i4", "i64": "<i8", "u8": "|u1", "bool": "|b1",
          "bf16": "<u2"}[entry["dtype"]]
    out = np.empty(tuple(e for _, e in ranges), dt)
    for coords in cells(ranges, w):
        loc = entry["chunks"][ckey(coords)]
        fname = os.path.join(root, *path.split("/"), f"process_{loc['p']}", *scoped.split("/"),
                             f"c.{ckey(coords)}")
        with open(fname, "rb") as f:
            chunk = np.frombuffer(f.read(), dt).reshape(w)
        cell = tuple((c * s, s) for c, s in zip(coords, w))
        hit = [(max(a, b), min(a + e, b + s) - max(a, b)) for (a, e), (b, s) in zip(ranges, cell)]
        src = tuple(slice(h - b, h - b + n) for (h, n), (b, _) in zip(hit, cell))
        dst = tuple(slice(h - a, h - a + n) for (h, n), (a, _) in zip(hit, ranges))
        out[dst] = chunk[src]
    return out


def restore_from_directory(root: str, path: str, processes: int) -> dict[str, np.ndarray]:
    """load_pipeline.py:406-493 on a per-leaf checkpoint saved with its own topology:
    each simulated process (one thread) reads its devices' shard ranges, then the global
    arrays are assembled."""
    import threading

    with open(os.path.join(root, *path.split("/"), "merged_index.json"), "rb") as f:
        arrays = json.loads(f.read())["arrays"]
    pieces: list[list] = [[] for _ in range(processes)]

    def work(p):
        for scoped, entry in arrays.items():
            sh = entry["sharding"]
            if sh is None:
                if p == 0:
                    whole = tuple((0, g) for g in entry["global_shape"])
                    pieces[p].append((scoped, whole, _read_range(root, path, scoped, entry, whole)))
                continue
            spec = Spec(Mesh([tuple(a) for a in sh["axes"]], processes), sh["spec"], sh["global_shape"])
            seen = set()
            for dev, ranges, _ in spec.shards():
                if spec.mesh.proc[dev] == p and ranges not in seen:
                    seen.add(ranges)
                    pieces[p].append((scoped, ranges, _read_range(root, path, scoped, entry, ranges)))

    threads = [threading.Thread(target=work, args=(p,)) for p in range(processes)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    out = {}
    for scoped, entry in arrays.items():
        dt = {"f32": "<f4", "bf16": "<u2"}.get(entry["dtype"], "<f8")
        out[scoped] = np.empty(tuple(entry["global_shape"]), dt)
    for plist in pieces:
        for scoped, ranges, data in plist:
            out[scoped][tuple(slice(o, o + e) for o, e in ranges)] = data
    return out
