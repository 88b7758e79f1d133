"""Host logic of the save's synchronous phase (CPU): the cyclic GC is paused for the
phase (nesting-safe across threads) and the caller's streams are captured on its own
thread (empty without a GPU)."""

from __future__ import annotations

import gc
import threading

from paper_2605_23066_b200 import save_pipeline as sp


def test_gc_paused_nests_and_restores():
    assert gc.isenabled()
    with sp._gc_paused():
        assert not gc.isenabled()
        with sp._gc_paused():
            assert not gc.isenabled()
        assert not gc.isenabled()
    assert gc.isenabled()


def test_gc_paused_across_threads():
    inside = threading.Event()
    release = threading.Event()

    def other():
        with sp._gc_paused():
            inside.set()
            release.wait(5)

    t = threading.Thread(target=other)
    t.start()
    inside.wait(5)
    with sp._gc_paused():
        assert not gc.isenabled()
    assert not gc.isenabled()  # the other thread's pause is still open
    release.set()
    t.join()
    assert gc.isenabled()


def test_gc_paused_keeps_a_disabled_collector_disabled():
    gc.disable()
    try:
        with sp._gc_paused():
            pass
        assert not gc.isenabled()
    finally:
        gc.enable()


def test_collect_behind_runs_a_pass_on_the_helper_thread_for_large_restores():
    import time

    from paper_2605_23066_b200 import gcpolicy

    c = gcpolicy._COLLECTOR
    before = c.passes
    with gcpolicy.paused():
        assert not gcpolicy.collect_behind(gcpolicy.COLLECT_BEHIND_BYTES - 1)  # too short to hide
        assert gcpolicy.collect_behind(gcpolicy.COLLECT_BEHIND_BYTES)
        deadline = time.time() + 10
        while c.passes == before and time.time() < deadline:
            time.sleep(0.01)
        assert c.passes > before
        assert not gc.isenabled()  # the pass does not re-enable the paused collector
    assert gc.isenabled()
    gc.disable()
    try:  # a caller that disabled the collector keeps it off: no passes behind its back
        with gcpolicy.paused():
            assert not gcpolicy.collect_behind(gcpolicy.COLLECT_BEHIND_BYTES)
    finally:
        gc.enable()


def test_caller_streams_without_gpu():
    class RT:
        gpus = [0]

    assert sp.caller_streams(RT()) == {}


def test_reference_defaults_switch_load_options():
    from paper_2605_23066_b200 import compat
    from paper_2605_23066_b200.load_pipeline import LoadOptions, reference_defaults

    assert LoadOptions().to_host is False and LoadOptions().read_once is True
    reference_defaults(True)
    try:
        assert compat.enabled()
        assert LoadOptions().to_host is True and LoadOptions().read_once is False
        assert LoadOptions(read_once=True).read_once is True  # explicit values still win
    finally:
        reference_defaults(False)
    assert LoadOptions().to_host is False


def test_restore_requests_the_gc_pass_when_its_last_thread_enters_the_engine(monkeypatch):
    """Threads runtime: every local restoring thread announces its engine call; only the
    last one requests the pass (an earlier request would stall the others' table
    building behind the GIL-holding collector)."""
    import types

    from paper_2605_23066_b200 import gcpolicy
    from paper_2605_23066_b200.load_pipeline import _RestoreJob

    calls = []
    monkeypatch.setattr(gcpolicy, "collect_behind", lambda n: calls.append(n) or True)
    job = types.SimpleNamespace(lock=threading.Lock(), engine_entries=0, engine_bytes=0,
                                local_processes={0, 1, 2},
                                items_by_process={0: ["a"], 1: ["b"], 2: [], 3: ["remote"]})
    _RestoreJob.entering_engine(job, 6 << 30)
    assert calls == []
    _RestoreJob.entering_engine(job, 2 << 30)
    assert calls == [4 << 30]  # mean bytes per busy local process
