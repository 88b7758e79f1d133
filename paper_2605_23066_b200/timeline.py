"""Per-process phase timelines of the most recent save / restore (instrumentation that
bench.py reports beside the throughput, so host-side overhead is visible per phase)."""

from __future__ import annotations

import gc
import time

_GC_MS = [0.0]  # Python garbage-collection time of this process so far (all threads)
_GC_START = [0.0]


def _gc_clock(phase, info) -> None:
    if phase == "start":
        _GC_START[0] = time.perf_counter()
    else:
        _GC_MS[0] += (time.perf_counter() - _GC_START[0]) * 1e3


gc.callbacks.append(_gc_clock)


class Timeline:
    """Wall-clock milliseconds spent in each phase, stamped at the end of the phase; a
    phase during which the process spent ≥ 0.5 ms collecting garbage also gets a
    ``<phase>.gc`` entry (part of the phase's time, not added to it)."""

    def __init__(self):
        self.t = time.perf_counter()
        self.gc = _GC_MS[0]
        self.phases: dict[str, float] = {}

    def stamp(self, phase: str) -> None:
        now = time.perf_counter()
        self.phases[phase] = round(self.phases.get(phase, 0.0) + (now - self.t) * 1e3, 3)
        self.t = now
        collected = _GC_MS[0] - self.gc
        self.gc = _GC_MS[0]
        if collected >= 0.5:
            key = phase + ".gc"
            self.phases[key] = round(self.phases.get(key, 0.0) + collected, 3)


# process index -> {phase: ms}; index -1 holds the calling thread's own phases
LAST_SAVE: dict[int, dict[str, float]] = {}
LAST_RESTORE: dict[int, dict[str, float]] = {}
