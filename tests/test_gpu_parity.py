"""Parity of the B200 data path with the reference (golden fixtures) and the oracle.

Every case of tests/golden/cases.py is saved through this package's public API from
device shards (ShardedArray on the GPU) and must produce exactly the files the real
reference produced (sha256 of every key).  Every listed load must put exactly
global[ranges] on every target device (oracle), and in reference-equivalent read mode
(read_once=False) read exactly the reference's per-process payload bytes; in read-once
mode each needed stored chunk is read exactly once.
"""

from __future__ import annotations

import json
import tempfile
from pathlib import Path

import numpy as np
import pytest

import cases
import helpers
import treevault_oracle as orc

pytestmark = pytest.mark.gpu

GOLDEN = Path(__file__).resolve().parent / "golden"


def fixture(name):
    return json.loads((GOLDEN / f"{name}.json").read_text())


@pytest.fixture(params=["default", "tiny_slots"])
def engine_cfg(request):
    from paper_2605_23066_b200 import native

    if request.param == "tiny_slots":
        # Forces payloads to be split across slots and strided boxes across pack batches.
        return native.EngineConfig(slot_bytes=4096, n_slots=3, staging_bytes=1 << 20, threads=3)
    return native.EngineConfig()


def _save(c, tmp, engine_cfg, sync=True):
    import paper_2605_23066_b200 as tv

    tree, specs = cases.build_inputs(c)
    backend = helpers.make_backend(c["backend"], tmp)
    rt = tv.SimulatedRuntime(c["process_count"], backend)
    rt.engine_config = engine_cfg
    cps = helpers.checkpointables(tree, specs, rt)
    opts = tv.SaveOptions(**c["options"], sync=sync)
    handle = tv.save_checkpoint(rt, "ckpt/run", cps, helpers.shardings_for(tree, specs), opts)
    handle.wait()
    return tree, specs, backend, rt


@pytest.mark.parametrize("name", [c["name"] for c in cases.CASES])
@pytest.mark.parametrize("sync", [True, False])
def test_save_matches_reference_bytes(name, sync, engine_cfg, tmp_path):
    c = cases.case(name)
    gold = fixture(name)
    _, _, backend, _ = _save(c, str(tmp_path), engine_cfg, sync=sync)
    got = helpers.dump_digests(backend)
    assert sorted(got) == sorted(gold["files"])
    for key, rec in gold["files"].items():
        assert got[key] == (rec["size"], rec["sha256"]), key
    # byte accounting per process identical to the reference (payload puts)
    for ident, rec in gold["save_counters"].items():
        if not ident.startswith("process_"):
            continue
        assert backend.counters(ident).payload_bytes_written == rec["payload_bytes_written"], ident


@pytest.mark.parametrize("name", [c["name"] for c in cases.CASES])
def test_load_matches_oracle(name, engine_cfg, tmp_path):
    import paper_2605_23066_b200 as tv

    c = cases.case(name)
    gold = fixture(name)
    tree, specs, backend, _ = _save(c, str(tmp_path), engine_cfg)
    for load, rec in zip(c["loads"], gold["loads"]):
        for read_once in ([load.get("read_once", True)] + ([True] if load.get("read_once") is False else [])):
            abstracts, mesh, P = helpers.abstracts_for(c, load, tree, specs)
            rt = tv.SimulatedRuntime(P, backend)
            rt.engine_config = engine_cfg
            before = {i: backend.counters(i) for i in backend.identities()}
            opts = tv.LoadOptions(broadcast=bool(load.get("broadcast")), read_once=read_once)
            if load.get("broadcast"):
                out = tv.load_with_broadcast(rt, "ckpt/run", abstracts, opts)
            else:
                out = tv.load_checkpoint(rt, "ckpt/run", abstracts, opts, current_mesh=mesh)
            for name_cp, value in tree.items():
                if not isinstance(value, dict):
                    continue
                for path, leaf in cases.leaf_paths(value):
                    got = helpers.get_path(out[name_cp], path)
                    if leaf[0] != "array":
                        continue
                    if isinstance(got, tv.ShardedArray):
                        spec = orc.Spec(orc.Mesh(*_mesh_args(got.sharding)), got.sharding.spec.entries,
                                        leaf[2].shape)
                        expect = orc.expected_shards(leaf[2], spec)
                    else:
                        expect = orc.expected_shards(leaf[2], None)
                    assert helpers.leaf_bytes_by_device(got) == expect, (load, path)
            if not read_once:
                for ident, counters in rec["counters"].items():
                    if not ident.startswith("process_"):
                        continue
                    now = backend.counters(ident)
                    prev = before.get(ident)
                    delta = now.minus(prev) if prev is not None else now
                    assert delta.payload_bytes_read == counters["payload_bytes_read"], (load, ident)


def _mesh_args(sharding):
    m = sharding.mesh
    return list(zip(m.axis_names, m.axis_sizes)), m.process_count, m.replica_axis


def test_read_once_reads_each_chunk_once(tmp_path):
    """Reshard 4-way FSDP -> (replica 2 x fsdp 2): every stored chunk is needed by two
    replicas; read-once reads the checkpoint's payload exactly once in total."""
    import paper_2605_23066_b200 as tv

    c = cases.case("fsdp4_per_leaf")
    tree, specs, backend, _ = _save(c, str(tmp_path), None)
    load = c["loads"][1]
    abstracts, mesh, P = helpers.abstracts_for(c, load, tree, specs)
    stored = sum(len(v) for k, v in backend.dump().items() if tv.backend.is_payload_key(k))
    before = backend.counters().payload_bytes_read
    rt = tv.SimulatedRuntime(P, backend)
    tv.load_checkpoint(rt, "ckpt/run", abstracts, tv.LoadOptions(read_once=True))
    assert backend.counters().payload_bytes_read - before == stored
