"""Random save / restore cases shared by the golden generator (real reference, build
container) and the GPU parity test: random meshes (1-3 axes, replica axis or not, 1-8
devices, processes = devices or fewer), random per-dimension specs, every dtype, both
layouts (small target files so packs span several data files), replica-parallel on and
off, subchunked read grids."""

from __future__ import annotations

import random

import numpy as np

import cases

N_CASES = 120

MESHES = [
    ([("fsdp", 2)], None), ([("fsdp", 4)], None), ([("fsdp", 8)], None),
    ([("replica", 2), ("fsdp", 2)], "replica"), ([("replica", 2), ("fsdp", 4)], "replica"),
    ([("replica", 4), ("fsdp", 2)], "replica"), ([("dp", 2), ("tp", 2)], None),
    ([("replica", 2), ("fsdp", 2), ("tp", 2)], "replica"),
]
DTYPES = ["f32", "bf16", "f64", "i32", "i64", "u8", "bool"]


def spec(rng, axes, P, ra, shape):
    names = [n for n, _ in axes if n != ra] + ([ra] if ra and rng.random() < 0.2 else [])
    sizes = dict(axes)
    entries, used = [], set()
    for g in shape:
        opts = [n for n in names if n not in used and g % sizes[n] == 0]
        pick = rng.choice(opts + [None] * 2) if opts else None
        if pick:
            used.add(pick)
        entries.append(pick)
    return (axes, P, ra, tuple(entries))


def case(seed):
    rng = random.Random(seed)
    nrng = np.random.default_rng(seed)
    axes, ra = rng.choice(MESHES)
    devices = int(np.prod([s for _, s in axes]))
    P = rng.choice([d for d in (devices, devices // 2, 1) if d >= 1 and devices % d == 0])
    tree, specs = {"m": {}}, {"m": {}}
    for i in range(rng.randint(1, 4)):
        rank = rng.randint(1, 3)
        shape = tuple(rng.choice([8, 16, 24, 32]) for _ in range(rank))
        dt = rng.choice(DTYPES)
        tree["m"][f"a{i}"] = cases.arr(nrng, dt, shape)
        if rng.random() < 0.85:
            specs["m"][f"a{i}"] = spec(rng, axes, P, ra, shape)
    options = {"layout": rng.choice(["per_leaf", "aggregated"]),
               "replica_parallel": bool(ra) and rng.random() < 0.6,
               "target_file_bytes": rng.choice([1 << 10, 4 << 10, 64 << 20])}
    if rng.random() < 0.4:
        options["subchunk_target_bytes"] = rng.choice([64, 256])
    return tree, specs, options, P, axes


def restore_targets(seed, tree, P):
    """A different random sharding (same process count) for each array of case ``seed``."""
    rng = random.Random(10_000 + seed)
    mesh_axes, ra = rng.choice([m for m in MESHES if int(np.prod([s for _, s in m[0]])) % P == 0])
    return {name: spec(rng, mesh_axes, P, ra, leaf[2].shape) for name, leaf in tree["m"].items()}
