"""The async save's blocking phase (reference: ``SaveSession.take_snapshot``,
``save_pipeline.py:308-326``; ownership contract ``save_pipeline.py:602-606``): after
``save_checkpoint`` returns the caller may mutate its arrays.

* the device snapshot is ordered on the CALLER's current stream, also when that is a
  side stream (``with torch.cuda.stream(s)``) and the runtime's worker threads sit on the
  default stream;
* when HBM cannot hold the snapshot arena the snapshot falls back to pinned host memory
  (forced here with TVGPU_SNAPSHOT=host) and the checkpoint stays byte-identical to the
  reference's (golden fixtures)."""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest

import cases
import helpers

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def test_snapshot_ordered_on_callers_side_stream(tmp_path):
    import torch

    import paper_2605_23066_b200 as tv

    backend = tv.FilesystemBackend(str(tmp_path))
    rt = tv.SimulatedRuntime(2, backend, gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 2)], process_count=2)
    shape = (4096, 4096)
    s = tv.Sharding(mesh, tv.PartitionSpec(("fsdp", None)), shape)
    g = torch.arange(shape[0] * shape[1], dtype=torch.float32, device="cuda:0").view(shape)
    want = g.cpu().numpy().copy()
    shards = {0: g[:2048].clone(), 1: g[2048:].clone()}
    leaf = tv.ShardedArray("f32", s, shards)
    torch.cuda.synchronize()
    side = torch.cuda.Stream(device=0)
    for i in range(3):
        # the default stream (the runtime workers' current stream) is held busy, so a
        # snapshot wrongly queued there would run after the side stream's update below
        torch.cuda._sleep(100_000_000)
        with torch.cuda.stream(side):
            h = tv.save_checkpoint(rt, f"ck{i}", {"m": {"w": leaf}}, {"m": {"w": s}}, tv.SaveOptions())
            for t in shards.values():
                t.add_(1.0)  # the next "optimizer step", on the caller's side stream
        h.wait()
        torch.cuda.synchronize()
        out = tv.load_checkpoint(rt, f"ck{i}", None, tv.LoadOptions(to_host=True), current_mesh=mesh)
        assert np.array_equal(out["m"]["w"].data, want + i), i


@pytest.mark.parametrize("name", ["fsdp4_per_leaf", "fsdp4_aggregated", "replica_parallel", "mixed_rename_agg"])
def test_host_snapshot_fallback_is_byte_identical(name, tmp_path, monkeypatch):
    import paper_2605_23066_b200 as tv

    names = [c["name"] for c in cases.CASES]
    if name not in names:
        pytest.skip(f"no golden case {name}")
    monkeypatch.setenv("TVGPU_SNAPSHOT", "host")
    c = cases.case(name)
    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    tree, specs = cases.build_inputs(c)
    backend = helpers.make_backend(c["backend"], str(tmp_path))
    rt = tv.SimulatedRuntime(c["process_count"], backend)
    cps = helpers.checkpointables(tree, specs, rt)
    handle = tv.save_checkpoint(rt, "ckpt/run", cps, helpers.shardings_for(tree, specs),
                                tv.SaveOptions(**c["options"], sync=False))
    kinds = {h.session.snapshot_kind for h in handle.handles} - {None}
    handle.wait()
    assert kinds <= {"host"} and kinds, kinds
    got = helpers.dump_digests(backend)
    assert sorted(got) == sorted(gold["files"])
    for key, rec in gold["files"].items():
        assert got[key] == (rec["size"], rec["sha256"]), key
