"""Saves that overwrite recycled files (engine side of the recycle pool): a checkpoint
retired with ``recycle=True`` hands its chunk files to the next save of the same tree,
which claims a file of each output's exact size and overwrites every byte.  The stored
checkpoint must still be byte-identical to the reference's (golden fixtures), the pool
must be consumed, and a Checkpointer(recycle=True) loop must keep exactly its retained
steps loadable."""

from __future__ import annotations

import json
from pathlib import Path

import pytest

import cases
import helpers

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


@pytest.mark.parametrize("name", ["fsdp4_per_leaf", "fsdp4_aggregated", "c1_per_leaf"])
def test_save_over_recycled_files_is_byte_identical(name, tmp_path):
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    c = cases.case(name)
    if c["backend"] != "fs":
        pytest.skip("recycling is a filesystem-backend feature")
    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    tree, specs = cases.build_inputs(c)
    backend = tv.FilesystemBackend(str(tmp_path))
    rt = tv.SimulatedRuntime(c["process_count"], backend)
    cps = helpers.checkpointables(tree, specs, rt)
    sh = helpers.shardings_for(tree, specs)
    opts = tv.SaveOptions(**c["options"])
    # a different checkpoint of the same tree, then retired into the pool
    tv.save_checkpoint(rt, "ckpt/old", cps, sh, opts).wait()
    delete_checkpoint(backend.store(), "ckpt/old", recycle=True)
    pooled = backend.recycle_pool_bytes()
    assert pooled > 0
    before = native.totals()["save"]["recycled_files"]
    tv.save_checkpoint(rt, "ckpt/run", cps, sh, opts).wait()
    assert native.totals()["save"]["recycled_files"] > before
    assert backend.recycle_pool_bytes() == 0  # every retired file was claimed
    got = helpers.dump_digests(backend)
    assert sorted(got) == sorted(gold["files"])
    for key, rec in gold["files"].items():
        assert got[key] == (rec["size"], rec["sha256"]), key


def test_checkpointer_recycle_loop(tmp_path):
    import numpy as np
    import torch

    import paper_2605_23066_b200 as tv

    backend = tv.FilesystemBackend(str(tmp_path))
    rt = tv.SimulatedRuntime(2, backend, gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 2)], process_count=2)
    s = tv.Sharding(mesh, tv.PartitionSpec(("fsdp", None)), (256, 128))
    shards = {0: torch.zeros(128, 128, device="cuda"), 1: torch.zeros(128, 128, device="cuda")}
    leaf = tv.ShardedArray("f32", s, shards)
    ck = tv.Checkpointer(rt, "run", tv.RetentionPolicy(keep_last=2), tv.SaveOptions(sync=False),
                         background_delete=True, recycle=True)
    for step in range(6):
        for t in shards.values():
            t.fill_(float(step))
        ck.save_step(step, {"m": {"w": leaf}}, {"m": {"w": s}})
    ck.close()  # joins the save and the background retention, drains the pool
    assert ck.all_steps() == [4, 5]
    assert backend.recycle_pool() is None
    for step in (4, 5):
        out = ck.load_step(step, options=tv.LoadOptions(to_host=True), current_mesh=mesh)
        assert np.all(out["m"]["w"].data == float(step))
