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


@pytest.fixture
def shm_dir(tmp_path):
    """A directory on a RAM-backed filesystem (the zero-copy half needs tmpfs)."""
    import shutil
    import uuid

    from paper_2605_23066_b200 import native

    d = f"/dev/shm/tv_recycle_{uuid.uuid4().hex[:8]}"
    yield d
    native.lib().tv_mapping_release_all()  # registrations of this test's files
    shutil.rmtree(d, ignore_errors=True)


@pytest.mark.parametrize("register", [True, False])
@pytest.mark.parametrize("name", ["fsdp4_per_leaf", "fsdp4_aggregated", "c1_per_leaf", "replica_parallel"])
def test_save_over_recycled_files_is_byte_identical(name, register, shm_dir, monkeypatch):
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    c = cases.case(name)
    if c["backend"] != "fs":
        pytest.skip("recycling is a filesystem-backend feature")
    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    tree, specs = cases.build_inputs(c)
    monkeypatch.setenv("TVGPU_SAVE_PATH", "zero_copy")  # (register=False: no zero-copy at all)
    monkeypatch.setenv("TVGPU_REGISTER_BUDGET", "1.0")  # register every first-claimed file
    backend = tv.FilesystemBackend(shm_dir, register_pool=register)
    rt = tv.SimulatedRuntime(c["process_count"], backend)
    cps = helpers.checkpointables(tree, specs, rt)
    sh = helpers.shardings_for(tree, specs)
    opts = tv.SaveOptions(**c["options"])
    # older checkpoints of the same tree, retired into the pool: the first claim of a
    # recycled file registers it (and writes it through the slot path... or zero-copy
    # right away), the second claim finds it registered
    tv.save_checkpoint(rt, "ckpt/old", cps, sh, opts).wait()
    delete_checkpoint(backend.store(), "ckpt/old", recycle=True)
    tv.save_checkpoint(rt, "ckpt/older", cps, sh, opts).wait()
    delete_checkpoint(backend.store(), "ckpt/older", recycle=True)
    pooled = backend.recycle_pool_bytes()
    assert pooled > 0
    before = native.totals()
    tv.save_checkpoint(rt, "ckpt/run", cps, sh, opts).wait()
    after = native.totals()
    assert after["save"]["recycled_files"] > before["save"]["recycled_files"]
    # registered pool: the chunk bytes went straight into the recycled files' pages
    zero_copy = after["save"]["zero_copy_bytes"] - before["save"]["zero_copy_bytes"]
    assert (zero_copy > 0) == register
    assert backend.recycle_pool_bytes() == 0  # every retired file was claimed
    got = helpers.dump_digests(backend)
    got = {k: v for k, v in got.items() if not k.startswith(".tvpool")}
    assert sorted(got) == sorted(gold["files"])
    for key, rec in gold["files"].items():
        assert got[key] == (rec["size"], rec["sha256"]), key
    # and a restore of it (zero-copy H2D out of the registered pages) is exact
    before = native.totals()
    abstracts, mesh, P = helpers.abstracts_for(c, {"mesh": "saved"}, tree, specs)
    out = tv.load_checkpoint(tv.SimulatedRuntime(P, backend), "ckpt/run", abstracts, tv.LoadOptions(),
                             current_mesh=mesh)
    if register:
        assert native.totals()["load"]["zero_copy_bytes"] > before["load"]["zero_copy_bytes"]
    for name_cp, value in tree.items():
        if not isinstance(value, dict):
            continue
        for path, leaf in cases.leaf_paths(value):
            if leaf[0] != "array":
                continue
            got_leaf = helpers.get_path(out[name_cp], path)
            if isinstance(got_leaf, tv.ShardedArray):
                import treevault_oracle as orc

                m = got_leaf.sharding.mesh
                spec = orc.Spec(orc.Mesh(list(zip(m.axis_names, m.axis_sizes)), m.process_count,
                                         m.replica_axis), got_leaf.sharding.spec.entries, leaf[2].shape)
                assert helpers.leaf_bytes_by_device(got_leaf) == orc.expected_shards(leaf[2], spec), path
            else:
                assert got_leaf.tobytes() == leaf[2].tobytes(), path


def test_checkpointer_recycle_loop(shm_dir, monkeypatch):
    import numpy as np
    import torch

    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native

    monkeypatch.setenv("TVGPU_SAVE_PATH", "zero_copy")
    monkeypatch.setenv("TVGPU_REGISTER_BUDGET", "1.0")
    backend = tv.FilesystemBackend(shm_dir, register_pool=True)
    rt = tv.SimulatedRuntime(2, backend, gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 2)], process_count=2)
    s = tv.Sharding(mesh, tv.PartitionSpec(("fsdp", None)), (256, 128))
    shards = {0: torch.zeros(128, 128, device="cuda"), 1: torch.zeros(128, 128, device="cuda")}
    leaf = tv.ShardedArray("f32", s, shards)
    ck = tv.Checkpointer(rt, "run", tv.RetentionPolicy(keep_last=2), tv.SaveOptions(sync=False),
                         background_delete=True, recycle=True)
    for step in range(10):  # step k reuses step k-3's files; registered from their 2nd claim
        for t in shards.values():
            t.fill_(float(step))
        ck.save_step(step, {"m": {"w": leaf}}, {"m": {"w": s}})
    ck.close()  # joins the save and the background retention, drains the pool
    assert ck.all_steps() == [8, 9]
    assert backend.recycle_pool(0) is None and backend.recycle_pool(1) is None
    assert native.totals()["save"]["zero_copy_bytes"] > 0
    for step in (8, 9):
        out = ck.load_step(step, options=tv.LoadOptions(to_host=True), current_mesh=mesh)
        assert np.all(out["m"]["w"].data == float(step))


@pytest.mark.parametrize("name", ["fsdp4_per_leaf", "replica_parallel", "fsdp4_aggregated"])
@pytest.mark.parametrize("path", ["zero_copy", "slots"])
def test_both_save_paths_over_recycled_files(path, name, shm_dir, monkeypatch):
    """The adaptive save-path choice may pick either path for a recycled save: both
    write the reference's bytes."""
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    monkeypatch.setenv("TVGPU_SAVE_PATH", path)
    monkeypatch.setenv("TVGPU_REGISTER_BUDGET", "1.0")
    c = cases.case(name)  # replica_parallel: strided segments, packed into the file (zero-copy)
    gold = json.loads((GOLDEN / f"{name}.json").read_text())
    tree, specs = cases.build_inputs(c)
    backend = tv.FilesystemBackend(shm_dir, register_pool=True)
    rt = tv.SimulatedRuntime(c["process_count"], backend)
    cps = helpers.checkpointables(tree, specs, rt)
    sh = helpers.shardings_for(tree, specs)
    for i in range(4):  # fresh, recycled (registered at this claim), then registered
        before = native.totals()["save"]
        tv.save_checkpoint(rt, "ckpt/run", cps, sh, tv.SaveOptions(**c["options"], sync=i % 2 == 0)).wait()
        after = native.totals()["save"]
        got = {k: v for k, v in helpers.dump_digests(backend).items() if not k.startswith(".tvpool")}
        assert got == {k: (r["size"], r["sha256"]) for k, r in gold["files"].items()}
        if i >= 2:
            zc = after["zero_copy_bytes"] - before["zero_copy_bytes"]
            assert (zc > 0) == (path == "zero_copy")
        delete_checkpoint(backend.store(), "ckpt/run", recycle=True)


def test_registrations_released_by_unlink_and_cold_restore(shm_dir, monkeypatch):
    """A checkpoint written zero-copy restores correctly after the process dropped every
    registration (a fresh process: pread path), and deleting it without recycling
    releases the registrations of its files."""
    import numpy as np
    import torch

    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    monkeypatch.setenv("TVGPU_SAVE_PATH", "zero_copy")
    monkeypatch.setenv("TVGPU_REGISTER_BUDGET", "1.0")
    native.lib().tv_mapping_release_all()
    backend = tv.FilesystemBackend(shm_dir, register_pool=True)
    rt = tv.SimulatedRuntime(1, backend, gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
    s = tv.Sharding(mesh, tv.PartitionSpec(("fsdp", None)), (1024, 1024))
    w = torch.randn(1024, 1024, device="cuda")
    leaf = tv.ShardedArray("f32", s, {0: w})
    for name in ("a", "b"):  # a: fresh; b: claims a's files and registers them
        tv.save_checkpoint(rt, name, {"m": {"w": leaf}}, {"m": {"w": s}}).wait()
        delete_checkpoint(backend.store(), name, recycle=True)
    before = native.totals()["save"]["zero_copy_bytes"]
    tv.save_checkpoint(rt, "c", {"m": {"w": leaf}}, {"m": {"w": s}}).wait()
    assert native.totals()["save"]["zero_copy_bytes"] > before
    files, nbytes = native.mapping_stats()
    assert files >= 1 and nbytes >= w.numel() * 4
    native.lib().tv_mapping_release_all()  # "a new process": nothing registered
    assert native.mapping_stats() == (0, 0)
    out = tv.load_checkpoint(rt, "c", None, tv.LoadOptions(to_host=True), current_mesh=mesh)
    assert np.array_equal(out["m"]["w"].data, w.cpu().numpy())
    # registered again by a save over recycled files, then freed by a plain delete
    delete_checkpoint(backend.store(), "c", recycle=True)
    tv.save_checkpoint(rt, "d", {"m": {"w": leaf}}, {"m": {"w": s}}).wait()
    assert native.mapping_stats()[0] >= 1
    delete_checkpoint(backend.store(), "d", recycle=False)
    assert native.mapping_stats() == (0, 0)
