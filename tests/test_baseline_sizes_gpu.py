"""Parity at BASELINE sizes: stored bytes and restored shards against the
oracle's independent restatement of the reference, not a round trip.

* C1 — 4 x (4096, 4096) f32 unsharded (268,435,456 bytes): every stored file of the
  per-leaf and aggregated layouts, sync and async, equals the oracle's
  ``expected_checkpoint`` (payloads = ``np.ascontiguousarray(data[sel]).tobytes()``,
  reference ``chunkstore.py:387-392``), including every metadata document.
* C3 — replica-parallel save on the (replica 2 x fsdp 4) mesh, P = 8, of every distinct
  leaf shape of the C2 tree at full size (one transformer layer + embed + lm_head +
  final_norm, bf16 params + f32 mu/nu: 12.7 GB).  These are the strided packs of the
  reference's replica segments (write chunks q/o (1024,2048), k/v (256,2048), gate/up
  (3584,2048), down (1024,7168), embed (16032,4096); Appendix B): every stored file's
  sha256 equals the oracle's; the single-slice save too.
* C4 — the same leaves saved 1 x 8 (FSDP-8, P = 8) and restored onto (replica 2 x fsdp 2)
  with P = 4 and onto (replica 2 x fsdp 4) with P = 8: every target shard equals
  ``global[ranges]`` (oracle ranges), compared on the device.

The 8 logical devices fold onto the GPUs present (threads runtime)."""

from __future__ import annotations

import hashlib
import os
import shutil

import numpy as np
import pytest

import treevault_oracle as orc

pytestmark = pytest.mark.gpu

D, FFN, VOCAB, KV = 4096, 14336, 128256, 1024
LAYER = {"attn/q": (D, D), "attn/k": (KV, D), "attn/v": (KV, D), "attn/o": (D, D),
         "mlp/gate": (FFN, D), "mlp/up": (FFN, D), "mlp/down": (D, FFN),
         "norm_in": (D,), "norm_post": (D,)}
SHAPES = {"embed": (VOCAB, D), "lm_head": (VOCAB, D), "final_norm": (D,),
          **{f"layers/0/{k}": v for k, v in LAYER.items()}}
TREES = (("params", "bf16"), ("mu", "f32"), ("nu", "f32"))


def _sha(b) -> str:
    return hashlib.sha256(b).hexdigest()


def _nest(flat: dict) -> dict:
    out: dict = {}
    for path, leaf in flat.items():
        node = out
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = leaf
    return out


def _globals(seed: int) -> dict:
    """Global host arrays of the sample, generated on the GPU (bf16 as uint16 bits)."""
    import torch

    gen = torch.Generator(device="cuda")
    out = {}
    for ti, (tree, dtype) in enumerate(TREES):
        for li, (path, shape) in enumerate(SHAPES.items()):
            gen.manual_seed(seed + 100 * ti + li)
            if dtype == "bf16":
                t = torch.randint(-32768, 32767, shape, dtype=torch.int16, device="cuda", generator=gen)
                out[(tree, path)] = ("bf16", t.cpu().numpy().view(np.uint16))
            else:
                t = torch.empty(shape, dtype=torch.float32, device="cuda").normal_(0, 1e-3, generator=gen)
                out[(tree, path)] = ("f32", t.cpu().numpy())
            del t
    torch.cuda.empty_cache()
    return out


def _stored_digests(root: str) -> dict:
    out = {}
    for dirpath, dirs, names in os.walk(root):
        if ".tvpool" in dirs:
            dirs.remove(".tvpool")  # the recycle pool holds no checkpoint files
        for n in names:
            full = os.path.join(dirpath, n)
            with open(full, "rb") as f:
                data = f.read()
            out[os.path.relpath(full, root).replace(os.sep, "/")] = (len(data), _sha(data))
    return out


def _compare_with_oracle(root: str, expected: dict) -> None:
    got = _stored_digests(root)
    want = {k: (len(v), _sha(v)) for k, v in expected.items()}
    assert sorted(got) == sorted(want), sorted(set(got) ^ set(want))[:10]
    bad = [k for k in want if got[k] != want[k]]
    assert bad == [], bad[:10]


def _fresh(path: str) -> str:
    shutil.rmtree(path, ignore_errors=True)
    os.makedirs(path)
    return path


def _gpus(n: int) -> list[int]:
    import torch

    return list(range(min(n, torch.cuda.device_count())))


@pytest.mark.parametrize("layout", ["per_leaf", "aggregated"])
@pytest.mark.parametrize("sync", [True, False])
def test_c1_at_size_matches_oracle(layout, sync):
    import paper_2605_23066_b200 as tv

    rng = np.random.default_rng(0)
    arrays = {f"a{i}": rng.standard_normal((4096, 4096), dtype=np.float32) for i in range(4)}
    root = _fresh("/dev/shm/tv_c1_at_size")
    try:
        backend = tv.FilesystemBackend(root)
        rt = tv.SimulatedRuntime(1, backend, gpus=[0])
        tree = {"model": {k: tv.device_put(tv.DenseArray("f32", v), None, rt) for k, v in arrays.items()}}
        tv.save_checkpoint(rt, "ck", tree, None, tv.SaveOptions(layout=layout, sync=sync)).wait()
        expected = orc.expected_checkpoint({"model": {k: ("array", "f32", v) for k, v in arrays.items()}},
                                           {}, {"layout": layout}, 1, "fs", path="ck")
        assert sum(len(v) for k, v in expected.items() if "/process_0/" in k and not k.endswith(".json")) \
            == 4 * 4096 * 4096 * 4
        _compare_with_oracle(root, expected)
        out = tv.load_checkpoint(rt, "ck", None, tv.LoadOptions(to_host=True))
        for k, v in arrays.items():
            assert out["model"][k].data.tobytes() == v.tobytes(), k
    finally:
        shutil.rmtree(root, ignore_errors=True)


@pytest.fixture(scope="module")
def sample():
    import torch

    from paper_2605_23066_b200 import native

    native.release_pool()
    torch.cuda.empty_cache()
    return _globals(seed=11)


def _sharded_tree(tv, rt, glob, axes, P, replica_axis):
    mesh = tv.Mesh.create(axes, process_count=P, replica_axis=replica_axis)
    trees, shardings = {}, {}
    for (tree, path), (dtype, data) in glob.items():
        shape = data.shape
        s = tv.Sharding(mesh, tv.PartitionSpec(("fsdp",) + (None,) * (len(shape) - 1)), shape)
        trees.setdefault(tree, {})[path] = tv.device_put(tv.DenseArray(dtype, data), s, rt)
        shardings[f"{tree}/{path}"] = s
    return {"state": {t: _nest(v) for t, v in trees.items()}}, {"state": shardings}


def _neutral(glob, axes, P, replica_axis):
    tree = {"state": {}}
    specs = {"state": {}}
    per_tree: dict = {}
    for (t, path), (dtype, data) in glob.items():
        per_tree.setdefault(t, {})[path] = ("array", dtype, data)
        specs["state"][f"{t}/{path}"] = (axes, P, replica_axis, ("fsdp",) + (None,) * (data.ndim - 1))
    tree["state"] = {t: _nest(v) for t, v in per_tree.items()}
    return tree, specs


@pytest.mark.parametrize("replica_parallel", [True, False])
def test_c3_replica_mesh_at_size_matches_oracle(sample, replica_parallel, monkeypatch):
    """Saved three times over recycled files (fresh; claimed + registered; zero-copy: the
    strided segments packed into the registered files); the last one is compared."""
    import torch

    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    monkeypatch.setenv("TVGPU_SAVE_PATH", "zero_copy")
    axes, P, ra = [("replica", 2), ("fsdp", 4)], 8, "replica"
    root = _fresh("/dev/shm/tv_c3_at_size")
    try:
        backend = tv.FilesystemBackend(root, register_pool=True)
        rt = tv.SimulatedRuntime(P, backend, gpus=_gpus(P))
        state, shardings = _sharded_tree(tv, rt, sample, axes, P, ra)
        opts = tv.SaveOptions(replica_parallel=replica_parallel, sync=True)
        for name in ("a", "b"):
            tv.save_checkpoint(rt, name, state, shardings, opts).wait()
            delete_checkpoint(backend.store(), name, recycle=True)
        before = native.totals()["save"]["zero_copy_bytes"]
        tv.save_checkpoint(rt, "ck", state, shardings, opts).wait()
        assert native.totals()["save"]["zero_copy_bytes"] > before
        del state
        torch.cuda.empty_cache()
        tree, specs = _neutral(sample, axes, P, ra)
        expected = orc.expected_checkpoint(tree, specs, {"replica_parallel": replica_parallel}, P, "fs",
                                           path="ck")
        if replica_parallel:  # the strided segments of Appendix B really are what is stored
            import json

            meta = json.loads(expected["ck/merged_index.json"])["arrays"]
            assert meta["state/params/layers/0/attn/q"]["write_chunk"] == [1024, 2048]
            assert meta["state/mu/layers/0/mlp/down"]["write_chunk"] == [1024, 7168]
            assert meta["state/nu/layers/0/attn/k"]["write_chunk"] == [256, 2048]
            assert meta["state/params/embed"]["write_chunk"] == [16032, 4096]
        _compare_with_oracle(root, expected)
    finally:
        native.lib().tv_mapping_release_all()
        shutil.rmtree(root, ignore_errors=True)


@pytest.mark.parametrize("target", ["2x2_P4", "2x4_P8"])
def test_c4_reshard_at_size_matches_oracle(sample, target):
    import torch

    import paper_2605_23066_b200 as tv

    root = _fresh("/dev/shm/tv_c4_at_size")
    try:
        backend = tv.FilesystemBackend(root)
        rt = tv.SimulatedRuntime(8, backend, gpus=_gpus(8))
        state, shardings = _sharded_tree(tv, rt, sample, [("fsdp", 8)], 8, None)
        tv.save_checkpoint(rt, "ck", state, shardings, tv.SaveOptions(sync=True)).wait()
        del state
        torch.cuda.empty_cache()
        fs = 2 if target == "2x2_P4" else 4
        P = 2 * fs
        axes = [("replica", 2), ("fsdp", fs)]
        mesh = tv.Mesh.create(axes, process_count=P, replica_axis="replica")
        abstract, specs = {}, {}
        for (t, path), (dtype, data) in sample.items():
            spec = ("fsdp",) + (None,) * (data.ndim - 1)
            abstract.setdefault(t, {})[path] = tv.AbstractLeaf(
                "array", data.shape, dtype, tv.Sharding(mesh, tv.PartitionSpec(spec), data.shape))
            specs[(t, path)] = orc.Spec(orc.Mesh(axes, P, "replica"), spec, data.shape)
        rrt = tv.SimulatedRuntime(P, backend, gpus=_gpus(P))
        before = backend.counters().payload_bytes_read
        out = tv.load_checkpoint(rrt, "ck", {"state": {t: _nest(v) for t, v in abstract.items()}},
                                 tv.LoadOptions())
        stored = sum(d.nbytes for _, d in sample.values())
        assert backend.counters().payload_bytes_read - before == stored  # read once
        flat = dict(tv.flatten(out["state"]))
        bad = []
        for (t, path), (dtype, data) in sample.items():
            leaf = flat[f"{t}/{path}"]
            ints = torch.int16 if dtype == "bf16" else torch.int32
            g = torch.from_numpy(data.view(np.int16 if dtype == "bf16" else np.int32))
            for dev, ranges, _ in specs[(t, path)].shards():
                want = g[tuple(slice(o, o + e) for o, e in ranges)]
                got = leaf.shards[dev].view(ints).cpu()
                if not torch.equal(got, want):
                    bad.append((t, path, dev))
        assert bad == []
    finally:
        shutil.rmtree(root, ignore_errors=True)
