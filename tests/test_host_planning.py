"""Host-side planning (no GPU): the integer rules every stored byte depends on.

Known-answer values are the reference's own frozen vectors (test_chunkstore.py:56-121,
test_sharding.py:143-178); property tests compare with brute-force restatements.
"""

from __future__ import annotations

import itertools
import math
import random

import numpy as np
import pytest

import paper_2605_23066_b200 as tv
from paper_2605_23066_b200 import chunkstore, save_pipeline
from paper_2605_23066_b200.errors import ChunkStoreError, ShardingError, DivisibilityError, TopologyError


@pytest.mark.parametrize("shape,dtype,target,expect", [
    ((64, 64), "f32", 4096, (16, 64)),
    ((8, 8), "f32", 4096, (8, 8)),
    ((16, 16), "f32", 32 << 20, (16, 16)),
    ((15,), "f32", 16, (1,)),
    ((15,), "f32", 32, (5,)),
    ((49,), "f64", 60, (7,)),
    ((1, 1), "f64", 8, (1, 1)),
])
def test_choose_chunk_shape_known_answers(shape, dtype, target, expect):
    assert tv.choose_chunk_shape(shape, dtype, target) == expect


def test_choose_chunk_shape_rejects_target_below_itemsize():
    with pytest.raises(ChunkStoreError):
        tv.choose_chunk_shape((4,), "f64", 4)


def test_choose_chunk_shape_properties():
    rng = random.Random(5)
    for _ in range(200):
        shape = tuple(rng.choice([1, 2, 3, 4, 6, 8, 12, 16, 60]) for _ in range(rng.randint(1, 3)))
        dtype = rng.choice(["f32", "f64", "i32", "u8", "bool", "bf16"])
        isz = tv.dtypes.itemsize(dtype) if hasattr(tv, "dtypes") else None
        from paper_2605_23066_b200.dtypes import itemsize

        isz = itemsize(dtype)
        target = rng.choice([isz, 16, 64, 256, 4096])
        got = tv.choose_chunk_shape(shape, dtype, target)
        assert all(s % c == 0 for s, c in zip(shape, got))
        grids = itertools.product(*[[d for d in range(1, s + 1) if s % d == 0] for s in shape])
        if any(math.prod(g) * isz <= target for g in grids):
            assert math.prod(got) * isz <= target
        else:
            assert got == (1,) * len(shape)


@pytest.mark.parametrize("shard,n,expect", [
    ((16, 16), 1, (16, 16)), ((1024,), 4, (256,)), ((10,), 4, (1,)), ((8, 4), 4, (2, 4)),
    ((4, 16), 2, (4, 8)),
])
def test_derive_write_chunk_known_answers(shard, n, expect):
    got = chunkstore.derive_write_chunk(shard, n)
    assert got == expect
    # every ceil-division segment boundary falls on a chunk boundary
    ax = tv.sharding.segment_axis(shard) if hasattr(tv, "sharding") else None
    from paper_2605_23066_b200.sharding import segment_axis

    ax = segment_axis(shard)
    step = -(-shard[ax] // n)
    for o in range(n):
        lo = min(o * step, shard[ax])
        assert lo % got[ax] == 0


def _shard(extent):
    mesh = tv.Mesh.create([("data", 1)], 1)
    return tv.shards_of(tv.Sharding(mesh, tv.PartitionSpec.of(None), (extent,)))[0]


def test_replica_segments_known_answers():
    assert tv.replica_segments(_shard(1024), 4, 1) == ((256, 256),)
    assert tv.replica_segments(_shard(77), 1, 0) == ((0, 77),)
    sizes = [0 if (s := tv.replica_segments(_shard(10), 4, o)) is None else s[0][1] for o in range(4)]
    assert sizes == [3, 3, 3, 1]
    mesh = tv.Mesh.create([("data", 1)], 1)
    shard = tv.shards_of(tv.Sharding(mesh, tv.PartitionSpec.of(None, None), (4, 16)))[0]
    assert tv.replica_segments(shard, 2, 0) == ((0, 4), (0, 8))
    with pytest.raises(ShardingError):
        tv.replica_segments(shard, 2, 2)


def _random_sharding(rng):
    shape, axes, entries, devices = [], [], [], 1
    for dim in range(rng.randint(1, 3)):
        s = rng.choice([1, 2, 4, 8, 12])
        shape.append(s)
        k = rng.choice([d for d in (1, 2, 4) if s % d == 0])
        if k > 1:
            axes.append((f"a{dim}", k))
            entries.append(f"a{dim}")
            devices *= k
        else:
            entries.append(None)
    if rng.random() < 0.5:
        axes.append(("rep", 2))
        devices *= 2
    if not axes:
        axes = [("solo", 1)]
    P = rng.choice([p for p in (1, 2, 4) if devices % p == 0])
    mesh = tv.Mesh.create(axes, P, "rep" if any(a == "rep" for a, _ in axes) else None)
    return tv.Sharding(mesh, tv.PartitionSpec(tuple(entries)), tuple(shape)), P


@pytest.mark.parametrize("replica_parallel", [False, True])
def test_write_pieces_tile_the_array_exactly_once(replica_parallel):
    rng = random.Random(11)
    for _ in range(150):
        s, P = _random_sharding(rng)
        boxes = []
        for p in range(P):
            for ranges, dev in save_pipeline.write_pieces_for_process(s, s.global_shape, p, replica_parallel):
                boxes.append(ranges)
                # the device that sources the piece holds it and lives on the process
                assert s.mesh.process_of(dev) == p
                holder = dict((sh.device, sh.ranges) for sh in tv.shards_of(s))[dev]
                assert all(ho <= o and o + e <= ho + he for (o, e), (ho, he) in zip(ranges, holder))
        counts = np.zeros(s.global_shape, np.int32)
        for r in boxes:
            counts[tuple(slice(o, o + e) for o, e in r)] += 1
        assert (counts == 1).all()


def test_storage_meta_replica_parallel_aligns_chunks():
    mesh = tv.Mesh.create([("replica", 2), ("fsdp", 4)], 8, "replica")
    s = tv.Sharding(mesh, tv.PartitionSpec.of("fsdp", None), (4096, 4096))
    leaf = tv.treemodel.AbstractLeaf("array", (4096, 4096), "bf16")
    meta = save_pipeline.storage_meta_for(leaf, s, tv.SaveOptions(replica_parallel=True))
    # q (4096,4096) on 2x4, replica-parallel -> (1024, 2048) chunks
    assert meta.shard_shape == (1024, 4096)
    assert meta.write_chunk == (1024, 2048)


def test_plan_fetches_whole_vs_subchunk():
    meta = chunkstore.ArrayStorageMetadata((256, 64), "f32", (16, 16), (16, 16), (4, 16), "per_leaf")
    entry = {"chunks": {f"{i}.{j}": {"p": 0} for i in range(16) for j in range(4)}}
    # a (4, 64) row band needs one (4,16) subchunk from each of 4 chunks
    f = chunkstore.plan_fetches("ck", "m/w", entry, meta, [((8, 4), (0, 64))])
    assert [x.nbytes for x in f] == [4 * 16 * 4] * 4
    assert all(x.op == "get_range" for x in f)
    # the union of four bands covering a chunk fetches the whole chunk once
    reqs = [((r, 4), (0, 64)) for r in (0, 4, 8, 12)]
    f = chunkstore.plan_fetches("ck", "m/w", entry, meta, reqs)
    assert [x.nbytes for x in f] == [16 * 16 * 4] * 4 and all(x.op == "get" for x in f)


def test_mesh_and_topology_validation():
    with pytest.raises(ShardingError):
        tv.Mesh.create([("a", 3)], 2)
    mesh = tv.Mesh.create([("a", 2)], 2)
    with pytest.raises(DivisibilityError):
        tv.Sharding(mesh, tv.PartitionSpec.of("a"), (3,)).check_divisible()
    with pytest.raises(TopologyError):
        tv.validate_topology(tv.sharding.describe_mesh(mesh) | {"devices": [1, 0]}, mesh)


def test_fs_listing_matches_full_walk(tmp_path):
    backend = tv.FilesystemBackend(tmp_path)
    store = backend.store()
    for key in ["a/ck/x", "a/ck/y/z", "a/ckx/w", "a/c", "b/ck/x", "a/ck.tmp.1/q"]:
        store.put(key, b"1")
    (tmp_path / "a" / "ck" / "p.partial").write_bytes(b"x")
    everything = sorted(k for k in backend._list(""))
    for prefix in ["", "a/", "a/ck/", "a/ck", "a/c", "b", "zz/", "a/ck/y/"]:
        assert backend._list(prefix) == [k for k in everything if k.startswith(prefix)], prefix


def test_box_index_matches_linear_scan():
    """BoxIndex (bisection on grid shardings) returns exactly the linear scan's hits, in
    input order, for mesh shardings (replicas included) and for arbitrary box sets."""
    import random

    from paper_2605_23066_b200 import chunkstore as cs
    from paper_2605_23066_b200.sharding import Mesh, PartitionSpec, Sharding, shards_of

    rng = random.Random(5)
    for case in range(300):
        rank = rng.randint(1, 3)
        shape = tuple(rng.choice([4, 8, 12, 16]) for _ in range(rank))
        if case % 3 == 2:  # arbitrary, possibly overlapping boxes
            boxes = []
            for _ in range(rng.randint(1, 6)):
                b = []
                for g in shape:
                    o = rng.randint(0, g - 1)
                    b.append((o, rng.randint(1, g - o)))
                boxes.append(tuple(b))
        else:
            axes = [("a", rng.choice([1, 2])), ("b", rng.choice([1, 2, 4]))]
            mesh = Mesh.create(axes, process_count=1)
            names = [None, "a", "b"]
            spec = [rng.choice(names) for _ in range(rank)]
            used = [n for n in spec if n]
            if len(used) != len(set(used)) or any(
                    g % dict(axes)[n] for g, n in zip(shape, spec) if n):
                continue
            boxes = [sh.ranges for sh in shards_of(Sharding(mesh, PartitionSpec.of(*spec), shape))]
        index = cs.BoxIndex(boxes)
        for _ in range(10):
            q = []
            for g in shape:
                o = rng.randint(0, g - 1)
                q.append((o, rng.randint(1, g - o)))
            q = tuple(q)
            expect = [i for i, b in enumerate(boxes) if cs._intersect(q, b) is not None]
            assert index.hits(q) == expect, (boxes, q)


def test_memoised_fetch_and_consumer_geometry():
    """The memoised fetch geometry bound to a leaf gives the same fetches as planning it
    from scratch, and the cached consumer geometry names exactly the boxes each fetch
    meets and, among them, those it lands in as one contiguous run."""
    import random

    from paper_2605_23066_b200 import chunkstore as cs
    from paper_2605_23066_b200 import load_pipeline as lp

    rng = random.Random(11)
    for case in range(200):
        rank = rng.randint(1, 3)
        w = tuple(rng.choice([2, 4, 8]) for _ in range(rank))
        r = tuple(wi // rng.choice([d for d in (1, 2, 4) if wi % d == 0]) for wi in w)
        g = tuple(wi * rng.randint(1, 3) for wi in w)
        meta = cs.ArrayStorageMetadata(g, "f32", g, w, r, "per_leaf")
        entry = {"chunks": {cs.coords_key(c): {"p": 0} for c in cs._covering(tuple((0, e) for e in g), w)}}
        reqs = []
        for _ in range(rng.randint(1, 4)):
            b = []
            for e in g:
                o = rng.randint(0, e - 1)
                b.append((o, rng.randint(1, e - o)))
            reqs.append(tuple(b))
        fetches = cs.plan_fetches("ck", f"t/l{case}", entry, meta, reqs)
        geometry = cs.fetch_geometry(w, r, 4, tuple(reqs))
        assert cs.fetches_at("ck", f"t/l{case}", entry, geometry) == fetches
        for f in fetches:
            assert f.key.startswith(f"ck/process_0/t/l{case}/c.")
        for f, (hits, direct) in zip(fetches, lp._consumer_geometry(geometry, tuple(reqs))):
            box = tuple(zip(f.origin, f.shape))
            assert list(hits) == [i for i, b in enumerate(reqs) if cs._intersect(box, b) is not None]
            expect = []
            for i in hits:
                b = reqs[i]
                inside = all(to <= bo and bo + be <= to + te for (bo, be), (to, te) in zip(box, b))
                if inside and cs.box_is_contiguous(tuple(e for _, e in b),
                                                   tuple(bo - to for (bo, _), (to, _) in zip(box, b)),
                                                   f.shape):
                    expect.append(i)
            assert list(direct) == expect


def test_numa_cpu_placement_from_sysfs(tmp_path):
    """The GPU's local CPUs come from its PCI device's local_cpulist, and only when the
    host has more than one NUMA node with CPUs (force: always)."""
    from paper_2605_23066_b200 import native

    assert native.parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert native.parse_cpulist("") == set()
    nodes = tmp_path / "devices" / "system" / "node"
    (nodes / "node0").mkdir(parents=True)
    (nodes / "node0" / "cpulist").write_text("0-15\n")
    dev = tmp_path / "bus" / "pci" / "devices" / "0000:1b:00.0"
    dev.mkdir(parents=True)
    (dev / "local_cpulist").write_text("16-31\n")
    assert native.numa_local_cpus("0000:1b:00.0", sysfs=str(tmp_path)) is None  # one node
    assert native.numa_local_cpus("0000:1b:00.0", sysfs=str(tmp_path), force=True) == set(range(16, 32))
    (nodes / "node1").mkdir()
    (nodes / "node1" / "cpulist").write_text("16-31\n")
    (nodes / "node2").mkdir()  # memory-only node: no CPUs
    (nodes / "node2" / "cpulist").write_text("\n")
    assert native.numa_local_cpus("0000:1b:00.0", sysfs=str(tmp_path)) == set(range(16, 32))
    assert native.numa_local_cpus("0000:99:00.0", sysfs=str(tmp_path)) is None  # unknown device


def test_bound_to_restores_affinity():
    import os

    from paper_2605_23066_b200 import native

    before = os.sched_getaffinity(0)
    one = {min(before)}
    with native._bound_to(one):
        assert os.sched_getaffinity(0) == one
    assert os.sched_getaffinity(0) == before
    with native._bound_to(None):
        assert os.sched_getaffinity(0) == before
