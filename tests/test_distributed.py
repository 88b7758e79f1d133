"""One-process-per-GPU runtime (torchrun), world size 2.

CPU (gloo): coordination — barriers, leader broadcast, step catalog, per-rank write plans.
GPU: the full data path across processes — byte-identical save from per-rank device
shards and an IPC-mapped read-once reshard restore (runs on 1 GPU with both ranks
sharing it, or on 2 GPUs).
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
WORKER = ROOT / "tests" / "dist_worker.py"


def _torchrun(mode: str, tmp: Path, port: int) -> subprocess.CompletedProcess:
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(WORKER), mode, str(tmp)]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    return subprocess.run(cmd, capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)


def test_coordination_world2_gloo(tmp_path):
    r = _torchrun("coord", tmp_path, 29531)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok") == 2


@pytest.mark.gpu
def test_datapath_world2(tmp_path):
    r = _torchrun("datapath", tmp_path, 29532)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok") == 2
