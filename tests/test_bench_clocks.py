"""bench.py's clock sampler (no GPU): only the job's GPUs count toward the clocks line.

nvidia-smi ignores CUDA_VISIBLE_DEVICES, so on a box with more GPUs than the job uses the
idle ones must be filtered out, by PCI address (UUIDs are redacted on some boxes).
"""

from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import bench  # noqa: E402


def _row(bus, sm, hw="Not Active"):
    return f"{bus}, {sm}, 1965, 300.0, 0x0, {hw}, Not Active, Not Active, Not Active\n"


def _sampler(tmp_path, rows, buses):
    c = bench.ClockSampler(0)
    c.path = str(tmp_path / "clk.csv")
    with open(c.path, "w") as f:
        f.writelines(rows)

    class _Done:
        def terminate(self): pass
        def wait(self): pass

    c.proc, c.f, c.buses = _Done(), open(os.devnull, "w"), set(buses)
    return c


def test_bus_parse():
    assert bench.ClockSampler._bus("00000000:D1:00.0") == (0, 0xD1, 0)
    assert bench.ClockSampler._bus("0000:1b:00.0") == (0, 0x1B, 0)
    assert bench.ClockSampler._bus("not a bus") is None


def test_idle_neighbours_filtered(tmp_path):
    rows = [_row("00000000:53:00.0", 1965), _row("00000000:D1:00.0", 120),
            _row("00000000:53:00.0", 1965), _row("00000000:D1:00.0", 120, hw="Active")]
    out = _sampler(tmp_path, rows, {(0, 0x53, 0)}).stop()
    assert out["sm_mhz"] == 1965 and out["samples"] == 2 and out["gpus_sampled"] == 1
    assert out["reasons"] == []


def test_unresolved_buses_sample_every_gpu(tmp_path):
    rows = [_row("00000000:53:00.0", 1965), _row("00000000:D1:00.0", 120, hw="Active")]
    out = _sampler(tmp_path, rows, {(0, 0x99, 0)}).stop()
    assert out["samples"] == 2 and out["gpus_sampled"] == "all"
    assert out["reasons"] == ["hw_slowdown"]
