"""Builders shared by the GPU tests: neutral case notation -> this package's objects."""

from __future__ import annotations

import hashlib
import tempfile
from pathlib import Path

import numpy as np

import cases
import paper_2605_23066_b200 as tv


def sharding(spec, shape):
    axes, P, replica_axis, entries = spec
    mesh = tv.Mesh.create(list(axes), process_count=P, replica_axis=replica_axis)
    return tv.Sharding(mesh, tv.PartitionSpec(tuple(entries)), tuple(shape))


def to_leaf(node, spec, runtime, on_device=True):
    if node[0] == "array":
        if not on_device:
            return tv.DenseArray(node[1], node[2])
        s = sharding(spec, node[2].shape) if spec is not None else None
        return tv.device_put(tv.DenseArray(node[1], node[2]), s, runtime)
    if node[0] == "scalar":
        return tv.Scalar(node[1], node[2])
    return tv.Text(node[1])


def to_tree(node, specs, runtime, prefix="", on_device=True):
    if isinstance(node, tuple) and node and node[0] in ("array", "scalar", "text"):
        return to_leaf(node, specs.get(prefix), runtime, on_device)
    if isinstance(node, dict):
        return {k: to_tree(v, specs, runtime, f"{prefix}/{k}" if prefix else k, on_device) for k, v in node.items()}
    items = [to_tree(v, specs, runtime, f"{prefix}/{i}" if prefix else str(i), on_device) for i, v in enumerate(node)]
    return tuple(items) if isinstance(node, tuple) else items


def checkpointables(tree, shard_specs, runtime, on_device=True):
    out = {}
    for name, value in tree.items():
        if isinstance(value, tuple) and value and value[0] == "json":
            out[name] = tv.JsonDocument(value[1])
        elif isinstance(value, tuple) and value and value[0] == "stateful":
            out[name] = tv.CountingIterator(value[1])
        else:
            out[name] = to_tree(value, shard_specs.get(name, {}), runtime, "", on_device)
    return out


def shardings_for(tree, shard_specs):
    out = {}
    for name, per in shard_specs.items():
        leaves = dict(cases.leaf_paths(tree[name]))
        out[name] = {p: sharding(s, leaves[p][2].shape) for p, s in per.items()}
    return out


def make_backend(kind: str, tmp: str):
    if kind == "fs":
        return tv.FilesystemBackend(tmp)
    if kind == "mem":
        return tv.MemoryBackend()
    return tv.MemoryBackend(supports_atomic_rename=True)


def sha(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()


def dump_digests(backend) -> dict:
    return {k: (len(v), sha(v)) for k, v in backend.dump().items()}


def abstracts_for(c, load, tree, shard_specs):
    """(abstracts or None, current_mesh, process_count) like gen_golden.run_load."""
    if load["mesh"] == "saved" and not load.get("broadcast"):
        any_spec = next((s for per in shard_specs.values() for s in per.values()), None)
        if any_spec is None:
            return None, None, c["process_count"]
        axes, P, ra, _ = any_spec
        return None, tv.Mesh.create(list(axes), process_count=P, replica_axis=ra), P
    P = c["process_count"]
    abstracts = {}
    for name, value in tree.items():
        if not isinstance(value, dict):
            continue
        flat = {}
        for path, leaf in cases.leaf_paths(value):
            if leaf[0] == "array":
                spec = cases.target_spec(c, load, path, leaf)
                if spec == "saved":
                    spec = shard_specs.get(name, {}).get(path)
                elif spec is not None:
                    P = spec[1]
                s = sharding(spec, leaf[2].shape) if spec is not None else None
                flat[path] = tv.AbstractLeaf("array", leaf[2].shape, leaf[1], s)
            elif leaf[0] == "scalar":
                flat[path] = tv.AbstractLeaf("scalar", dtype=leaf[1])
            else:
                flat[path] = tv.AbstractLeaf("text")
        skel = tv.TreeStructureDoc.from_tree(to_tree(value, {}, None, "", on_device=False))
        abstracts[name] = skel.reconstruct(flat.__getitem__)
    return abstracts, None, P


def get_path(node, path):
    for part in path.split("/"):
        node = node[int(part)] if isinstance(node, (list, tuple)) else node[part]
    return node


def leaf_bytes_by_device(leaf) -> dict:
    """device id -> host bytes of a loaded leaf (ShardedArray) or {-1: bytes}."""
    if isinstance(leaf, tv.ShardedArray):
        return {d: tv.DenseArray(leaf.dtype, t).tobytes() for d, t in leaf.shards.items()}
    return {-1: leaf.tobytes()}
