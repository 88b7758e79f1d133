"""Test configuration: the `gpu` marker and shared helpers.

`-m "not gpu"` runs here (no GPU): oracle vs golden fixtures, host planning logic, the
C-ABI surface.  `-m gpu` runs on a B200 through `gpurun`: parity of the native data path
against the golden fixtures and the oracle.
"""

from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
sys.path.insert(0, str(ROOT / "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200) and libtvgpu.so")


def gpu_available() -> bool:
    try:
        import torch
    except ImportError:
        return False
    return torch.cuda.is_available()
