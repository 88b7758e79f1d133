"""Generate the golden fixtures by running the REAL reference (treevault) in this
container.  The reference is not available on the GPU box, so its outputs travel as the
small JSON files next to this script.

    python tests/golden/gen_golden.py            # rewrites tests/golden/*.json

For every case of cases.py: save with the reference on its own backend, record every
stored key (length + sha256, full text for JSON/COMMIT), the per-identity byte/op
counters, then run each listed load and record the per-identity counters and the sha256
of every loaded global array.  bf16 is not in the reference's dtype table
(dtypes.py:14-21); the documented shim registers it as its 2-byte bit pattern ("<u2").
"""

from __future__ import annotations

import hashlib
import json
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REFERENCE_SRC = Path("/root/reference/pkg/src")
sys.path.insert(0, str(HERE))

import cases  # noqa: E402


def _import_reference():
    if not REFERENCE_SRC.exists():
        raise SystemExit("the reference is only available in the build container")
    sys.path.insert(0, str(REFERENCE_SRC))
    import treevault
    import treevault.dtypes

    treevault.dtypes.NUMPY_DTYPES["bf16"] = np.dtype("<u2")  # SURVEY §0 shim
    return treevault


def to_reference(tv, node):
    if isinstance(node, tuple) and node and node[0] == "array":
        return tv.DenseArray(node[1], node[2])
    if isinstance(node, tuple) and node and node[0] == "scalar":
        return tv.Scalar(node[1], node[2])
    if isinstance(node, tuple) and node and node[0] == "text":
        return tv.Text(node[1])
    if isinstance(node, dict):
        return {k: to_reference(tv, v) for k, v in node.items()}
    if isinstance(node, tuple):
        return tuple(to_reference(tv, v) for v in node)
    return [to_reference(tv, v) for v in node]


def checkpointables(tv, tree):
    out = {}
    for name, value in tree.items():
        if isinstance(value, tuple) and value and value[0] == "json":
            out[name] = tv.JsonDocument(value[1])
        elif isinstance(value, tuple) and value and value[0] == "stateful":
            out[name] = tv.CountingIterator(value[1])
        else:
            out[name] = to_reference(tv, value)
    return out


def sharding(tv, spec, shape):
    axes, P, replica_axis, entries = spec
    mesh = tv.Mesh.create(list(axes), process_count=P, replica_axis=replica_axis)
    return tv.Sharding(mesh, tv.PartitionSpec(tuple(entries)), tuple(shape))


def make_backend(tv, kind, tmp):
    if kind == "fs":
        return tv.FilesystemBackend(tmp)
    if kind == "mem":
        return tv.MemoryBackend()
    return tv.MemoryBackend(supports_atomic_rename=True)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def run_case(tv, c) -> dict:
    tree, shard_specs = cases.build_inputs(c)
    arrays = {}
    for name, value in tree.items():
        if isinstance(value, dict):
            for path, leaf in cases.leaf_paths(value):
                if leaf[0] == "array":
                    arrays[(name, path)] = leaf
    shardings = {
        name: {p: sharding(tv, s, arrays[(name, p)][2].shape) for p, s in per.items()}
        for name, per in shard_specs.items()
    }
    with tempfile.TemporaryDirectory() as tmp:
        backend = make_backend(tv, c["backend"], tmp)
        rt = tv.SimulatedRuntime(c["process_count"], backend)
        opts = tv.SaveOptions(**c["options"])
        tv.save_checkpoint(rt, "ckpt/run", checkpointables(tv, tree), shardings, opts).wait()
        dump = backend.dump()
        files = {}
        for key, data in sorted(dump.items()):
            rec = {"size": len(data), "sha256": sha(data)}
            if key.endswith(".json") or key.endswith("COMMIT"):
                rec["text"] = data.decode("utf-8")
            files[key] = rec
        save_counters = {i: backend.counters(i).to_json() for i in backend.identities()}
        loads = []
        for load in c["loads"]:
            loads.append(run_load(tv, c, load, backend, tree, arrays, shardings))
    return {"case": c["name"], "files": files, "save_counters": save_counters, "loads": loads}


def run_load(tv, c, load, backend, tree, arrays, shardings) -> dict:
    before = {i: backend.counters(i) for i in backend.identities()}
    mesh_spec = load["mesh"]
    opts = tv.LoadOptions(broadcast=bool(load.get("broadcast")))
    if mesh_spec == "saved" and not load.get("broadcast"):
        any_s = next((s for per in shardings.values() for s in per.values()), None)
        mesh = any_s.mesh if any_s is not None else None
        P = mesh.process_count if mesh is not None else c["process_count"]
        rt = tv.SimulatedRuntime(P, backend)
        out = tv.load_checkpoint(rt, "ckpt/run", None, opts, current_mesh=mesh)
    else:
        abstracts = {}
        P = c["process_count"]
        for name, value in tree.items():
            if not isinstance(value, dict):
                abstracts[name] = None
                continue
            flat = {}
            for path, leaf in cases.leaf_paths(value):
                if leaf[0] == "array":
                    spec = cases.target_spec(c, load, path, leaf)
                    if spec == "saved":
                        s = shardings[name].get(path)
                    elif spec is None:
                        s = None
                    else:
                        s = sharding(tv, spec, leaf[2].shape)
                        P = spec[1]
                    flat[path] = tv.AbstractLeaf("array", leaf[2].shape, leaf[1], s)
                elif leaf[0] == "scalar":
                    flat[path] = tv.AbstractLeaf("scalar", dtype=leaf[1])
                else:
                    flat[path] = tv.AbstractLeaf("text")
            skeleton = tv.TreeStructureDoc.from_tree(to_reference(tv, value))
            abstracts[name] = skeleton.reconstruct(flat.__getitem__)
        abstracts = {k: v for k, v in abstracts.items() if v is not None}
        rt = tv.SimulatedRuntime(P, backend)
        out = tv.load_checkpoint(rt, "ckpt/run", abstracts, opts)
    counters = {}
    for ident in backend.identities():
        now = backend.counters(ident)
        prev = before.get(ident)
        counters[ident] = (now.minus(prev) if prev is not None else now).to_json()
    digests = {}
    for (name, path), leaf in arrays.items():
        node = out[name]
        for part in path.split("/"):
            node = node[int(part)] if isinstance(node, (list, tuple)) else node[part]
        got = node.data.tobytes()
        assert got == leaf[2].tobytes(), f"reference round trip differs at {name}/{path}"
        digests[f"{name}/{path}"] = sha(got)
    return {"load": load, "process_count": P, "counters": counters, "arrays": digests}


def cast_fixture(tv) -> dict:
    """The reference's cast_leaf (treemodel.py:444-484) on every numeric dtype pair."""
    out = []
    for src, dst, kind in cases.cast_cases():
        x = cases.cast_input(src, dst, kind)
        rec = {"src": src, "dst": dst, "kind": kind}
        try:
            got = tv.cast_leaf(tv.DenseArray(src, x), tv.AbstractLeaf("array", x.shape, dst))
            rec["sha256"] = sha(got.data.tobytes())
        except tv.TreevaultError as exc:
            rec["error"] = type(exc).__name__
            rec["message"] = str(exc)
        out.append(rec)
    return {"casts": out}


def main() -> None:
    tv = _import_reference()
    (HERE / "casts.json").write_text(json.dumps(cast_fixture(tv), indent=1, sort_keys=True))
    for c in cases.CASES:
        fixture = run_case(tv, c)
        (HERE / f"{c['name']}.json").write_text(json.dumps(fixture, indent=1, sort_keys=True))
        print(c["name"], len(fixture["files"]), "files")


if __name__ == "__main__":
    main()
