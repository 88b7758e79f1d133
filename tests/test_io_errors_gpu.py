"""Storage failures on the native path surface like the reference's: a save that runs out
of space on a real filesystem raises BackendError from wait(), leaves no finalized
checkpoint (the temp location is cleaned, no `.partial` residue), and a later save of a
fitting tree to the same path succeeds; a restore of a truncated chunk file raises
CorruptionError.  Needs root to mount a tiny tmpfs (skipped otherwise)."""

from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture
def tiny_tmpfs(tmp_path):
    mnt = tmp_path / "tiny"
    mnt.mkdir()
    rc = subprocess.run(["mount", "-t", "tmpfs", "-o", "size=4m", "tmpfs", str(mnt)],
                        capture_output=True).returncode
    if rc != 0:
        pytest.skip("cannot mount a tmpfs here (needs root)")
    try:
        yield mnt
    finally:
        subprocess.run(["umount", "-l", str(mnt)], capture_output=True)


def test_enospc_save_fails_cleanly_then_recovers(tiny_tmpfs):
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200.errors import BackendError

    backend = tv.FilesystemBackend(str(tiny_tmpfs))
    rt = tv.SimulatedRuntime(1, backend)
    big = np.arange(3 * 1024 * 1024, dtype=np.float32).reshape(3, 1024, 1024)  # 12 MiB > 4 MiB
    for sync in (True, False):
        h = tv.save_checkpoint(rt, f"ck{int(sync)}", {"m": {"w": tv.device_put(tv.DenseArray("f32", big), None, rt)}},
                               None, tv.SaveOptions(sync=sync))
        with pytest.raises(BackendError):
            h.wait()
        assert not tv.save_pipeline.is_finalized(backend.store(), f"ck{int(sync)}")
        left = [os.path.join(d, f) for d, _, fs in os.walk(tiny_tmpfs) for f in fs]
        assert left == [], left  # temp location cleaned, no .partial residue
    small = np.arange(64 * 1024, dtype=np.float32)
    tv.save_checkpoint(rt, "ck1", {"m": {"w": tv.device_put(tv.DenseArray("f32", small), None, rt)}},
                       None, tv.SaveOptions(sync=True)).wait()
    out = tv.load_checkpoint(rt, "ck1", None, tv.LoadOptions(to_host=True))
    assert out["m"]["w"].tobytes() == small.tobytes()


def test_truncated_chunk_raises_corruption(tmp_path):
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200.errors import CorruptionError

    backend = tv.FilesystemBackend(str(tmp_path))
    rt = tv.SimulatedRuntime(1, backend)
    w = np.arange(4096, dtype=np.float32).reshape(64, 64)
    tv.save_checkpoint(rt, "ck", {"m": {"w": tv.device_put(tv.DenseArray("f32", w), None, rt)}},
                       None, tv.SaveOptions(sync=True)).wait()
    chunk = next(os.path.join(d, f) for d, _, fs in os.walk(tmp_path) for f in fs if f.startswith("c."))
    with open(chunk, "r+b") as f:
        f.truncate(100)
    with pytest.raises(CorruptionError):
        tv.load_checkpoint(rt, "ck")
