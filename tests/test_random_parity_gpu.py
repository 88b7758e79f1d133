"""Randomised save parity on the GPU path (tests/golden/random_cases.py: random meshes,
specs, dtypes, layouts with small target files, replica-parallel, subchunked reads; sync
and async saves): every stored file's length + sha256 equals what the REAL reference
wrote for the same inputs (tests/golden/random_cases.json, gen_random_golden.py).  Each
case then restores onto another random sharding — read-once and reference-equivalent —
and every target shard must equal global[ranges]; the reference-equivalent reads must read
exactly the reference's per-process payload bytes."""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import pytest

import helpers
import random_cases
import treevault_oracle as orc

pytestmark = pytest.mark.gpu

GOLDEN = json.loads((Path(__file__).resolve().parent / "golden" / "random_cases.json").read_text())


@pytest.mark.parametrize("seed", range(random_cases.N_CASES))
def test_random_save_matches_reference_and_restores(seed, tmp_path):
    import paper_2605_23066_b200 as tv

    tree, specs, options, P, _ = random_cases.case(seed)
    backend = tv.FilesystemBackend(str(tmp_path))
    rt = tv.SimulatedRuntime(P, backend)
    cps = helpers.checkpointables(tree, specs, rt)
    sync = seed % 2 == 0
    tv.save_checkpoint(rt, "ck/run", cps, helpers.shardings_for(tree, specs),
                       tv.SaveOptions(**options, sync=sync)).wait()
    got = {k: [len(v), hashlib.sha256(v).hexdigest()] for k, v in backend.dump().items()}
    want = GOLDEN[str(seed)]["files"]
    assert sorted(got) == sorted(want), (seed, sorted(set(got) ^ set(want))[:5])
    for k in want:
        assert got[k] == want[k], (seed, k)

    targets = random_cases.restore_targets(seed, tree, P)
    abstract = {name: tv.AbstractLeaf("array", leaf[2].shape, leaf[1], helpers.sharding(targets[name], leaf[2].shape))
                for name, leaf in tree["m"].items()}
    # read-once (default) and the reference-equivalent reads, whose per-process payload
    # bytes must equal what the reference read for the same restore
    for read_once in (True, False):
        before = {i: backend.counters(i) for i in backend.identities()}
        out = tv.load_checkpoint(rt, "ck/run", {"m": abstract}, tv.LoadOptions(read_once=read_once))
        for name, leaf in tree["m"].items():
            axes_t, P_t, ra_t, entries = targets[name]
            expect = orc.expected_shards(leaf[2], orc.Spec(orc.Mesh(axes_t, P_t, ra_t), entries, leaf[2].shape))
            for dev, t in out["m"][name].shards.items():
                assert tv.DenseArray(leaf[1], t).tobytes() == expect[dev], (seed, read_once, name, dev)
        if not read_once:
            for ident, nbytes in GOLDEN[str(seed)]["load_payload_bytes_read"].items():
                now, prev = backend.counters(ident), before.get(ident)
                delta = now.minus(prev) if prev is not None else now
                assert delta.payload_bytes_read == nbytes, (seed, ident)
