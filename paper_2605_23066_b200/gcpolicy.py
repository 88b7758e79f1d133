"""Keeping Python's cyclic garbage collector off the checkpoint's critical path.

A gen-2 pass over a training process's heap costs tens of milliseconds (measured inside
restore planning: 38-42 ms of a 47-55 ms phase, ``profiles/r02_gc_sources_n{2,4}.json``).
The save's synchronous phase and the restore's planning run with the collector paused
(``paused``); a large restore then has the pending collection run on a helper thread
while the calling threads wait in the native engine (``collect_behind``, requested right
before the blocking engine call by the last local restoring thread to get there,
``_RestoreJob.entering_engine``: the pass holds the GIL, so any Python work after the
request waits for it), so the pass overlaps the DMA instead of preceding it
(``profiles/r02_ab_gc_policy_n{1,4}.jsonl``)."""

from __future__ import annotations

import gc
import os
import threading

# a restore whose engine phase moves at least this many bytes per process hides a full
# collection behind its DMA (tens of ms at ≥ 40 GB/s)
COLLECT_BEHIND_BYTES = 4 << 30


def restore_policy_enabled() -> bool:
    """``TVGPU_GC_POLICY=0`` leaves restores to the interpreter's own schedule (A/B)."""
    return os.environ.get("TVGPU_GC_POLICY", "1") != "0"


class paused:
    """Collector disabled inside the block.  Nesting-safe across threads: the collector
    is re-enabled when the last pause ends, and only if it was enabled when the first
    began."""

    _lock = threading.Lock()
    _depth = 0
    _was_enabled = False

    def __enter__(self):
        with paused._lock:
            if paused._depth == 0:
                paused._was_enabled = gc.isenabled()
                gc.disable()
            paused._depth += 1
        return self

    def __exit__(self, *exc):
        with paused._lock:
            paused._depth -= 1
            if paused._depth == 0 and paused._was_enabled:
                gc.enable()


class _Collector:
    """One daemon thread per process running ``gc.collect()`` on request; requests
    arriving while a pass runs coalesce into the next one."""

    def __init__(self):
        self._lock = threading.Lock()
        self._wake = threading.Event()
        self._thread: threading.Thread | None = None
        self.passes = 0

    def request(self) -> None:
        with self._lock:
            if self._thread is None or not self._thread.is_alive():
                self._thread = threading.Thread(target=self._run, name="tv-gc-behind", daemon=True)
                self._thread.start()
        self._wake.set()

    def _run(self) -> None:
        while True:
            self._wake.wait()
            self._wake.clear()
            gc.collect()
            self.passes += 1


_COLLECTOR = _Collector()


def collect_behind(nbytes: int) -> bool:
    """Ask for a full collection on the helper thread when the native call about to
    start moves ``nbytes`` (long enough to hide it); returns whether one was requested.
    Only meaningful while the collector is ``paused`` — otherwise the interpreter
    collects on its own schedule anyway."""
    if nbytes < COLLECT_BEHIND_BYTES or paused._depth == 0 or not paused._was_enabled:
        return False
    _COLLECTOR.request()
    return True
