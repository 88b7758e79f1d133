"""Device-memory lifetime: a restore's HBM arena is released as soon as the caller drops
the result, and an async save's snapshot arena as soon as the save completes — by
reference counting, with the cyclic garbage collector disabled (a cycle holding either
arena would pin a tree-sized buffer until the next full collection: OOM at scale)."""

from __future__ import annotations

import gc

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_arenas_released_without_gc(tmp_path):
    import torch

    import paper_2605_23066_b200 as tv

    rt = tv.SimulatedRuntime(2, tv.FilesystemBackend(str(tmp_path)), gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 2)], process_count=2)
    rng = np.random.default_rng(3)
    tree, shardings = {}, {}
    for i in range(4):
        w = rng.standard_normal((256, 128)).astype(np.float32)
        s = tv.Sharding(mesh, tv.PartitionSpec.of("fsdp", None), w.shape)
        tree[f"w{i}"] = tv.device_put(tv.DenseArray("f32", w), s, rt)
        shardings[f"w{i}"] = s
    torch.cuda.synchronize()
    base = torch.cuda.memory_allocated(0)
    gc.collect()
    gc.disable()
    try:
        for step in range(2):
            h = tv.save_checkpoint(rt, f"ck{step}", {"m": tree}, {"m": shardings},
                                   tv.SaveOptions(sync=False))
            h.wait()
            del h
            assert torch.cuda.memory_allocated(0) == base, "snapshot arena outlived the save"
            out = tv.load_checkpoint(rt, f"ck{step}", None, tv.LoadOptions(), current_mesh=mesh)
            assert torch.cuda.memory_allocated(0) > base
            del out
            assert torch.cuda.memory_allocated(0) == base, "restore arena outlived its result"
    finally:
        gc.enable()
