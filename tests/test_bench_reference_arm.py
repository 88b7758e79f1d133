"""The reference arm of bench.py on CPU: the UNMODIFIED reference (staged in oracle/_ref by
oracle/ref_recipe.py) runs through its own public API on a tiny sample, and both arms
print the same ``config`` object (the driver compares them)."""

from __future__ import annotations

import argparse
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def _args(**kw):
    base = dict(config="c2", cpu_layers=0, layers=32, save_mode="async", layout="per_leaf", storage="shm",
                restore_gpus=None, dir="/dev/shm/tvbench_test")
    base.update(kw)
    return argparse.Namespace(**base)


def test_reference_leg_runs_the_unmodified_reference(tmp_path):
    import bench

    sys.path.insert(0, str(ROOT / "oracle"))
    import ref_recipe

    if not ref_recipe.available():
        pytest.skip("oracle/_ref not staged")
    res = bench.reference_leg(_args(), str(tmp_path), steps=1, warmup=0)
    assert res["kind"] == "reference" and res["value"] >= 0  # (GB/s of a 40 KB sample rounds to ~0)
    assert res["sample_bytes"] == 4096 * (2 + 4 + 4)  # final_norm of params (bf16) + mu + nu (f32)
    assert res["implementation"].startswith("treevault (unmodified")
    port = bench.port_leg(_args(), str(tmp_path))
    assert port["kind"] == "port" and port["sample_bytes"] == res["sample_bytes"]


def test_both_arms_print_the_same_config():
    import bench

    for cfg in ("c1", "c2", "c3", "c4"):
        a = bench.bench_config(_args(config=cfg), 8)
        b = bench.bench_config(_args(config=cfg), 8)
        assert a == b and a["config"] == cfg
    assert bench.bench_config(_args(), 1)["tree_bytes"] == bench.TREE_BYTES_C2
