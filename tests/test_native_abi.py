"""The C-ABI boundary without a GPU: libtvgpu.so loads, exports every function
include/tvgpu.h declares, and the ctypes/numpy descriptor layouts equal the C structs."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_header_symbol():
    from paper_2605_23066_b200 import native

    header = (ROOT / "include" / "tvgpu.h").read_text()
    declared = set(re.findall(r"^\s*(?:int|int64_t)\s+(tv_\w+)\s*\(", header, re.M))
    assert declared == set(native.EXPORTS)
    lib = native.lib()
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(native.LIB_PATH)],
                         capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (tv_\w+)", out))
    assert declared <= exported
    assert lib.tv_abi_version() == 2


def test_struct_layouts_match_numpy_dtypes(tmp_path):
    from paper_2605_23066_b200 import native

    exe = tmp_path / "abi_layout"
    subprocess.run(["gcc", "-std=c99", f"-I{ROOT / 'include'}", str(ROOT / "tests/native/abi_layout.c"),
                    "-o", str(exe)], check=True)
    lines = dict(l.rsplit(" ", 1) for l in subprocess.run([str(exe)], capture_output=True, text=True,
                                                           check=True).stdout.split("\n") if l)
    sizes = {"tv_array_box": native.ARRAY_BOX, "tv_copy": native.COPY, "tv_write_item": native.WRITE_ITEM,
             "tv_output": native.OUTPUT, "tv_read_item": native.READ_ITEM, "tv_input": native.INPUT,
             "tv_stats": native.STATS}
    for name, dt in sizes.items():
        assert int(lines[name]) == dt.itemsize, name
    for key, value in lines.items():
        if "." not in key:
            continue
        struct, field = key.split(".")
        assert sizes[struct].fields[field][1] == int(value), key


def test_last_error_reports_bad_arguments():
    from paper_2605_23066_b200 import native

    lib = native.lib()
    rc = lib.tv_engine_save(None, None, 0, None, 0, None)
    assert rc == -3
    assert "bad arguments" in native.last_error()


def test_no_gpu_means_loud_failure():
    """The product path refuses to run without CUDA (no CPU fallback)."""
    import torch

    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.errors import NativeError

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(NativeError):
        native.require_gpu()


def test_engine_sizing_rules(monkeypatch):
    """Measured sizing (profiles/r01_ab_slot_*.txt, r01_ab_threads_*.txt): one engine
    owning the host gets 4 MiB slots and cores - 1 storage threads; engines sharing the host
    split the cores (one kept for the producer only at >= 8 each) and use <= 2 MiB slots;
    2 slots per thread (>= 16)."""
    from paper_2605_23066_b200 import native

    monkeypatch.delenv("LOCAL_WORLD_SIZE", raising=False)
    for k in ("TVGPU_SLOT_BYTES", "TVGPU_SLOTS", "TVGPU_STAGING_BYTES", "TVGPU_THREADS"):
        monkeypatch.delenv(k, raising=False)
    monkeypatch.setattr(native, "_host_cores", lambda: 16)
    n_slots, slot, staging, threads = native.EngineConfig().sizing(1)
    assert (slot, threads, n_slots) == (4 << 20, 15, 30) and staging >= n_slots * slot
    n_slots, slot, staging, threads = native.EngineConfig().sizing(4)
    assert threads == 4 and slot <= 2 << 20 and n_slots == 16  # 4 cores each: no producer core
    monkeypatch.setattr(native, "_host_cores", lambda: 32)
    assert native.EngineConfig().sizing(4)[3] == 7                 # 8 cores each: one for the producer
    monkeypatch.setattr(native, "_host_cores", lambda: 16)
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "4")
    assert native.EngineConfig().sizing(1) == native.EngineConfig().sizing(4)
    monkeypatch.setenv("TVGPU_SLOT_BYTES", str(1 << 20))
    assert native.EngineConfig().sizing(1)[1] == 1 << 20


def test_unlink_many(tmp_path):
    """Native bulk unlink (no GPU needed): removed / absent flags; other errors raise."""
    from paper_2605_23066_b200 import native
    from paper_2605_23066_b200.errors import BackendError

    files = [tmp_path / f"f{i}" for i in range(50)]
    for f in files:
        f.write_bytes(b"x" * 100)
    got = native.unlink_many([str(f) for f in files] + [str(tmp_path / "missing")], 8)
    assert got == [True] * 50 + [False]
    assert not any(f.exists() for f in files)
    (tmp_path / "d").mkdir()
    with pytest.raises(BackendError):
        native.unlink_many([str(tmp_path / "d")], 2)
