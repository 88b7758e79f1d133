"""torchrun worker for the one-process-per-GPU runtime (tests/test_distributed.py).

    torchrun --nproc-per-node 2 tests/dist_worker.py <mode> <dir>

mode "coord" (CPU, gloo): barriers, leader broadcast, step catalog, per-rank write plans.
mode "datapath" (GPU): save the fsdp case from device shards on 2 ranks, compare every
stored file with the oracle, then reshard-restore onto (replica 2 x fsdp 1) through the
IPC-mapped read-once fan-out and compare every local shard with the oracle.
Exit code 0 = pass.
"""

from __future__ import annotations

import datetime
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def coord(base: str) -> None:
    import torch.distributed as dist

    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200 import save_pipeline

    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=90))  # fail, never hang
    backend = tv.FilesystemBackend(base)
    rt = tv.DistributedRuntime(backend, barrier_timeout=90.0)
    rank, world = rt.rank, rt.process_count
    ctx = rt.local
    ctx.barrier("a")
    got = ctx.leader_broadcast("nonce", b"abc" if rank == 0 else None)
    assert got == b"abc", got
    if rank == 0:
        for step, final in ((1, True), (2, True), (3, False)):
            store = backend.store()
            store.put(f"run/step_{step:08d}/x", b"1")
            if final:
                store.put(f"run/step_{step:08d}/global_metadata.json", b"{}")
    ctx.barrier("written")
    ck = tv.Checkpointer(rt, "run")
    assert ck.all_steps() == [1, 2], ck.all_steps()
    assert tv.latest_step(rt, "run") == 2
    # per-rank write plan: each rank persists exactly its own shards
    mesh = tv.Mesh.create([("fsdp", world)], process_count=world)
    s = tv.Sharding(mesh, tv.PartitionSpec.of("fsdp", None), (8 * world, 4))
    pieces = save_pipeline.write_pieces_for_process(s, s.global_shape, rank, False)
    assert pieces == [(((8 * rank, 8), (0, 4)), rank)], pieces
    gathered = rt.all_gather_object(pieces)
    assert len(gathered) == world
    # one Checkpointer per rank: retention deletes happen once (process 0), every rank's
    # catalog agrees, no rank sees another's deletion as a failure
    for background in (False, True):
        root = f"loop_{int(background)}"
        ck = tv.Checkpointer(rt, root, tv.RetentionPolicy(keep_last=2), tv.SaveOptions(sync=False),
                             background_delete=background)
        for step in range(5):
            ck.save_step(step, {"m": {"step": tv.Scalar("i64", step)}})
        ck.close()
        assert ck.all_steps() == [3, 4], ck.all_steps()
        ctx.barrier(f"loop{background}")
        assert sorted(tv.Checkpointer(rt, root).all_steps()) == [3, 4]
        got = ck.load_step()
        assert got["m"]["step"] == tv.Scalar("i64", 4)
    # a job of fewer logical processes than ranks (restore onto fewer GPUs): every rank
    # creates the subgroup, only its members get a runtime
    sub = tv.DistributedRuntime.subgroup(backend, [0], barrier_timeout=90.0)
    if rank == 0:
        assert sub is not None and sub.process_count == 1 and sub.rank == 0
        sub.local.barrier("sub")
        assert sub.local.leader_broadcast("sub-nonce", b"x") == b"x"
        assert sub.all_gather_object(7) == [7]
    else:
        assert sub is None
    ctx.barrier("done")
    dist.destroy_process_group()


def datapath(base: str) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    import cases
    import paper_2605_23066_b200 as tv
    import treevault_oracle as orc

    local = int(os.environ.get("LOCAL_RANK", "0"))
    gpu = local % torch.cuda.device_count()
    torch.cuda.set_device(gpu)
    dist.init_process_group("gloo", timeout=datetime.timedelta(seconds=90))  # fail, never hang
    backend = tv.FilesystemBackend(base)
    rt = tv.DistributedRuntime(backend, gpu=gpu, barrier_timeout=90.0)
    world = rt.process_count
    rng = np.random.default_rng(3)
    tree = {"state": cases.llama_like(rng, layers=1, d=32, ffn=48, vocab=40, kv=8)}
    specs = {"state": cases.fsdp_shardings(tree["state"], [("fsdp", world)], world)}
    # one unsharded leaf: process 0 writes it; on restore every rank receives a copy
    tree["state"]["extra"] = {"bias": cases.arr(rng, "f64", (6, 5))}
    leaves = dict(cases.leaf_paths(tree["state"]))
    shardings, state = {}, {}
    for path, leaf in leaves.items():
        spec = specs["state"].get(path)
        s = None
        if spec is not None:
            axes, P, ra, entries = spec
            mesh = tv.Mesh.create(list(axes), process_count=P, replica_axis=ra)
            s = tv.Sharding(mesh, tv.PartitionSpec(tuple(entries)), leaf[2].shape)
            shardings[path] = s
        node = state
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = tv.device_put(tv.DenseArray(leaf[1], leaf[2]), s, rt)
    for sync in (True, False):
        path = f"ck/run_{int(sync)}"
        tv.save_checkpoint(rt, path, {"state": state}, {"state": shardings},
                           tv.SaveOptions(sync=sync)).wait()
        rt.local.barrier(f"saved{sync}")
        if rt.rank == 0:
            expect = orc.expected_checkpoint(tree, specs, {}, world, "fs", path=path)
            got = backend.dump()
            got = {k: v for k, v in got.items() if k.startswith(path + "/")}
            assert sorted(got) == sorted(expect), sorted(set(got) ^ set(expect))
            for k, v in expect.items():
                assert got[k] == v, k
    # reshard restore onto (replica world x fsdp 1): every chunk needed by every rank
    mesh2 = tv.Mesh.create([("replica", world), ("fsdp", 1)], process_count=world, replica_axis="replica")
    abstract = {}
    for path, leaf in leaves.items():
        s2 = None if path.startswith("extra/") else tv.Sharding(
            mesh2, tv.PartitionSpec(("fsdp",) + (None,) * (leaf[2].ndim - 1)), leaf[2].shape)
        node = abstract
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = tv.AbstractLeaf("array", leaf[2].shape, leaf[1], s2)
    before = backend.counters(f"process_{rt.rank}").payload_bytes_read
    out = tv.load_checkpoint(rt, "ck/run_1", {"state": abstract})
    read = backend.counters(f"process_{rt.rank}").payload_bytes_read - before
    total_read = rt.all_gather_object(read)
    stored = sum(leaf[2].nbytes for leaf in leaves.values())
    assert sum(total_read) == stored, (total_read, stored)   # read once across ranks
    for path, leaf in leaves.items():
        node = out["state"]
        for p in path.split("/"):
            node = node[p]
        if path.startswith("extra/"):  # unsharded: a full copy on this rank's GPU
            assert isinstance(node, tv.DenseArray) and node.on_device
            assert node.tobytes() == leaf[2].tobytes(), path
            continue
        assert sorted(node.shards) == [rt.rank], node.shards.keys()
        got = tv.DenseArray(leaf[1], node.shards[rt.rank]).tobytes()
        assert got == leaf[2].tobytes(), path
    from paper_2605_23066_b200 import timeline

    assert "ipc_publish" in timeline.LAST_RESTORE[rt.rank]  # replicas: ranks write to each other
    # same sharding as saved (sharded leaves only: the unsharded one fans out from process
    # 0): every chunk lands in its reader's own process -> no IPC at all
    same_abs = {}
    for path, leaf in leaves.items():
        if path.startswith("extra/"):
            continue
        node = same_abs
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = tv.AbstractLeaf("array", leaf[2].shape, leaf[1], shardings[path])
    out = tv.load_checkpoint(rt, "ck/run_0", {"state": same_abs}, tv.LoadOptions(mode="partial"))
    assert "ipc_publish" not in timeline.LAST_RESTORE[rt.rank], timeline.LAST_RESTORE[rt.rank]
    for path, leaf in leaves.items():
        if path.startswith("extra/"):
            continue
        node = out["state"]
        for p in path.split("/"):
            node = node[p]
        ranges = dict((sh.device, sh.ranges) for sh in tv.shards_of(shardings[path]))[rt.rank]
        sel = tuple(slice(o, o + e) for o, e in ranges)
        got = tv.DenseArray(leaf[1], node.shards[rt.rank]).tobytes()
        assert got == np.ascontiguousarray(leaf[2][sel]).tobytes(), path
    # fused cast across processes: f32 leaves restored as f64 onto the replica mesh (the
    # reader's kernel converts while storing into the peer's arena)
    cast_abs = {}
    for path, leaf in leaves.items():
        if leaf[1] != "f32":
            continue
        node = cast_abs
        parts = path.split("/")
        for p in parts[:-1]:
            node = node.setdefault(p, {})
        node[parts[-1]] = tv.AbstractLeaf("array", leaf[2].shape, "f64", tv.Sharding(
            mesh2, tv.PartitionSpec(("fsdp",) + (None,) * (leaf[2].ndim - 1)), leaf[2].shape))
    out = tv.load_checkpoint(rt, "ck/run_1", {"state": cast_abs}, tv.LoadOptions(mode="partial"))
    n_cast = 0
    for path, leaf in leaves.items():
        if leaf[1] != "f32":
            continue
        node = out["state"]
        for p in path.split("/"):
            node = node[p]
        got = tv.DenseArray("f64", node.shards[rt.rank]).tobytes()
        assert got == leaf[2].astype(np.float64).tobytes(), path
        n_cast += 1
    assert n_cast > 0
    # restore onto FEWER processes than saved it (FSDP-world -> FSDP-1 on rank 0 only):
    # the torchrun shape of "saved on 8, restored onto 4"
    sub = tv.DistributedRuntime.subgroup(backend, [0], gpu=gpu, barrier_timeout=90.0)
    if sub is not None:
        mesh1 = tv.Mesh.create([("fsdp", 1)], process_count=1)
        one_abs = {}
        for path, leaf in leaves.items():
            if path.startswith("extra/"):
                continue
            node = one_abs
            parts = path.split("/")
            for p in parts[:-1]:
                node = node.setdefault(p, {})
            node[parts[-1]] = tv.AbstractLeaf("array", leaf[2].shape, leaf[1], tv.Sharding(
                mesh1, tv.PartitionSpec(("fsdp",) + (None,) * (leaf[2].ndim - 1)), leaf[2].shape))
        out = tv.load_checkpoint(sub, "ck/run_1", {"state": one_abs}, tv.LoadOptions(mode="partial"))
        for path, leaf in leaves.items():
            if path.startswith("extra/"):
                continue
            node = out["state"]
            for p in path.split("/"):
                node = node[p]
            assert tv.DenseArray(leaf[1], node.shards[0]).tobytes() == leaf[2].tobytes(), path
    rt.local.barrier("done")
    dist.destroy_process_group()


if __name__ == "__main__":
    mode, base = sys.argv[1], sys.argv[2]
    {"coord": coord, "datapath": datapath}[mode](base)
    print(f"rank {os.environ.get('RANK')} ok")
