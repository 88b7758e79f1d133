"""Per-process phase timelines of the most recent save / restore (instrumentation that
bench.py reports beside the throughput, so host-side overhead is visible per phase)."""

from __future__ import annotations

import time


class Timeline:
    """Wall-clock milliseconds spent in each phase, stamped at the end of the phase."""

    def __init__(self):
        self.t = time.perf_counter()
        self.phases: dict[str, float] = {}

    def stamp(self, phase: str) -> None:
        now = time.perf_counter()
        self.phases[phase] = round(self.phases.get(phase, 0.0) + (now - self.t) * 1e3, 3)
        self.t = now


# process index -> {phase: ms}; index -1 holds the calling thread's own phases
LAST_SAVE: dict[int, dict[str, float]] = {}
LAST_RESTORE: dict[int, dict[str, float]] = {}
