"""Recycle pool of the filesystem backend (host side, CPU): retention deletes with
``recycle=True`` retire chunk payload files into ``<root>/.tvpool/<size>/`` (metadata
documents are unlinked), the pool is invisible to listings and reserved as a key, and
``drain_recycle_pool`` frees it.  The engine side (saves overwriting pooled files) is
tests/test_recycle_gpu.py."""

from __future__ import annotations

import os

import pytest

import paper_2605_23066_b200 as tv
from paper_2605_23066_b200.errors import BackendError
from paper_2605_23066_b200.training_manager import delete_checkpoint


def _checkpoint(store, prefix):
    store.put(f"{prefix}/global_metadata.json", b"{}")
    store.put(f"{prefix}/process_0/array_metadata.json", b"{}")
    store.put(f"{prefix}/process_0/m/w/c.0.0", b"x" * 4096)
    store.put(f"{prefix}/process_0/m/w/c.1.0", b"y" * 4096)
    store.put(f"{prefix}/process_0/d/0", b"z" * 1000)


def test_recycle_retires_payloads_and_hides_the_pool(tmp_path):
    backend = tv.FilesystemBackend(tmp_path)
    store = backend.store()
    _checkpoint(store, "run/step_00000001")
    assert backend.recycle_pool() is None
    delete_checkpoint(store, "run/step_00000001", recycle=True)
    assert store.list_keys("") == []
    pool = backend.recycle_pool(0)  # files of process_0 go to its own sub-pool
    assert pool is not None and pool.endswith(os.path.join(".tvpool", "p0"))
    assert backend.recycle_pool(1) is None
    sizes = sorted((d, len(os.listdir(os.path.join(pool, d)))) for d in os.listdir(pool))
    assert sizes == [("1000", 1), ("4096", 2)]  # payload files only, grouped by size
    assert backend.recycle_pool_bytes() == 2 * 4096 + 1000
    assert not (tmp_path / "run" / "step_00000001").exists()  # emptied dirs pruned
    with pytest.raises(BackendError):
        store.put(".tvpool/x", b"1")
    assert backend.drain_recycle_pool() == 2 * 4096 + 1000
    assert backend.recycle_pool(0) is None


def test_plain_delete_frees(tmp_path):
    backend = tv.FilesystemBackend(tmp_path)
    store = backend.store()
    _checkpoint(store, "ck")
    delete_checkpoint(store, "ck")
    assert backend.recycle_pool(0) is None and store.list_keys("") == []


def test_memory_backend_ignores_recycle():
    backend = tv.MemoryBackend()
    store = backend.store()
    _checkpoint(store, "ck")
    delete_checkpoint(store, "ck", recycle=True)
    assert store.list_keys("") == [] and backend.recycle_pool(0) is None


def test_process_of_key():
    from paper_2605_23066_b200.chunkstore import process_of_key

    assert process_of_key("run/step_00000001/process_3/state/w/c.0.0") == 3
    assert process_of_key("ck/process_12/d/0") == 12
    assert process_of_key("ck/global_metadata.json") is None


def test_save_path_chooser_explores_then_exploits(monkeypatch):
    from paper_2605_23066_b200.native import SavePathChooser

    monkeypatch.delenv("TVGPU_SAVE_PATH", raising=False)
    c = SavePathChooser()
    key = (0, 37)
    assert c.choose(key) is True                      # explore zero-copy first
    c.record(key, True, 10 << 30, 1.0, warm_up=True)  # registered new files: not scored
    assert c.choose(key) is True
    c.record(key, True, 15 << 30, 1.0, warm_up=False)  # first touch of new registrations: not scored
    assert c.choose(key) is True
    c.record(key, True, 50 << 30, 1.0, warm_up=False)
    assert c.choose(key) is False                     # then the slot path
    c.record(key, False, 30 << 30, 1.0, warm_up=False)
    assert all(c.choose(key) for _ in range(3 * c.RETRY))  # clear winner: never re-tried
    # another save size on the same GPU follows the GPU's verdict without exploring
    assert c.choose((0, 33)) is True
    # a close call is re-tried once every RETRY saves
    close = (2, 37)
    c.record(close, True, 50 << 30, 1.0, warm_up=False)  # (discarded: first zero-copy sample)
    c.record(close, True, 50 << 30, 1.0, warm_up=False)
    c.record(close, False, 45 << 30, 1.0, warm_up=False)
    picks = [c.choose(close) for _ in range(c.RETRY)]
    assert picks.count(False) == 1
    assert c.choose((1, 37)) is True                  # another GPU explores on its own
    monkeypatch.setenv("TVGPU_SAVE_PATH", "slots")
    assert c.choose(key) is False
