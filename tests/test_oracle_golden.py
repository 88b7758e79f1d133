"""The oracle restatement is pinned against the real reference's outputs.

tests/golden/*.json were produced by running the reference (tests/golden/gen_golden.py);
here the numpy restatement in oracle/ must reproduce every stored file byte-for-byte
(sha256) and the reference's per-process chunk-payload read counters.
"""

from __future__ import annotations

import hashlib
import json
from pathlib import Path

import pytest

import cases
import treevault_oracle as orc

GOLDEN = Path(__file__).resolve().parent / "golden"


def fixture(name: str) -> dict:
    return json.loads((GOLDEN / f"{name}.json").read_text())


@pytest.mark.parametrize("name", [c["name"] for c in cases.CASES])
def test_oracle_reproduces_reference_checkpoint(name):
    c = cases.case(name)
    gold = fixture(name)
    tree, specs = cases.build_inputs(c)
    files = orc.expected_checkpoint(tree, specs, c["options"], c["process_count"], c["backend"])
    assert sorted(files) == sorted(gold["files"])
    for key, rec in gold["files"].items():
        data = files[key]
        assert len(data) == rec["size"], key
        if "text" in rec:
            assert data.decode("utf-8") == rec["text"], key
        assert hashlib.sha256(data).hexdigest() == rec["sha256"], key


def _metas(files: dict[str, bytes]) -> dict:
    merged = json.loads(files["ckpt/run/merged_index.json"])
    return {k: {kk: v[kk] for kk in ("global_shape", "dtype", "write_chunk", "read_chunk")}
            for k, v in merged["arrays"].items()}


def _target_specs(c, load, tree, specs):
    out = {}
    for name, value in tree.items():
        if not isinstance(value, dict):
            continue
        for path, leaf in cases.leaf_paths(value):
            if leaf[0] != "array":
                continue
            t = cases.target_spec(c, load, path, leaf)
            if t == "saved":
                t = specs.get(name, {}).get(path)
            if t is not None:
                axes, P, ra, entries = t
                t = orc.Spec(orc.Mesh(axes, P, ra), entries, leaf[2].shape)
            out[f"{name}/{path}"] = t
    return out


@pytest.mark.parametrize("name", [c["name"] for c in cases.CASES])
def test_oracle_reproduces_reference_read_counters(name):
    c = cases.case(name)
    gold = fixture(name)
    tree, specs = cases.build_inputs(c)
    files = orc.expected_checkpoint(tree, specs, c["options"], c["process_count"], c["backend"])
    metas = _metas(files)
    for load, rec in zip(c["loads"], gold["loads"]):
        targets = _target_specs(c, load, tree, specs)
        expect = orc.reference_read_bytes(tree, metas, targets, rec["process_count"],
                                          bool(load.get("broadcast")))
        for p, nbytes in expect.items():
            got = rec["counters"].get(f"process_{p}", {}).get("payload_bytes_read", 0)
            assert got == nbytes, (load, p)


def test_oracle_shard_bytes_match_reference_digests():
    c = cases.case("fsdp4_per_leaf")
    gold = fixture("fsdp4_per_leaf")
    tree, _ = cases.build_inputs(c)
    for scoped, digest in gold["loads"][0]["arrays"].items():
        name, path = scoped.split("/", 1)
        leaf = dict(cases.leaf_paths(tree[name]))[path]
        got = orc.expected_shards(leaf[2], None)[-1]
        assert hashlib.sha256(got).hexdigest() == digest


def test_oracle_reproduces_reference_on_random_cases():
    """The oracle's stored bytes equal the real reference's on 120 random save cases
    (random meshes / specs / dtypes / layouts / replica-parallel / subchunking)."""
    import hashlib

    import random_cases

    golden = json.loads((GOLDEN / "random_cases.json").read_text())
    assert len(golden) == random_cases.N_CASES
    for seed in range(random_cases.N_CASES):
        tree, specs, options, P, _ = random_cases.case(seed)
        files = orc.expected_checkpoint(tree, specs, options, P, "fs", path="ck/run")
        got = {k: [len(v), hashlib.sha256(v).hexdigest()] for k, v in files.items()}
        assert got == golden[str(seed)]["files"], seed
