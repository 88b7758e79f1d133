"""Storage-side probe: is writing a checkpoint's bytes into FRESH tmpfs files slower than
overwriting pages that already exist (page allocation + kernel zeroing on the critical
path)?  pwrite from a 4 MiB buffer, T threads, each writing its own files:

  fresh      create + pwrite (what a save does today)
  overwrite  pwrite over the same files again (pages already allocated)
  renamed    files renamed to new names first, then overwritten (a recycled file)

    python tools/recycle_probe.py <dir> [threads] [GiB per thread]
"""

from __future__ import annotations

import json
import os
import sys
import threading
import time

import numpy as np


def run(d, threads, per_thread, mode, names):
    block = 4 << 20
    buf = np.random.default_rng(0).integers(0, 255, block, dtype=np.uint8)
    mv = memoryview(buf)
    files_per = max(1, per_thread // (64 << 20))
    fsize = per_thread // files_per

    def work(t):
        for f in range(files_per):
            name = names(t, f)
            flags = os.O_WRONLY | os.O_CREAT | (os.O_TRUNC if mode == "fresh" else 0)
            fd = os.open(name, flags, 0o644)
            off = 0
            while off < fsize:
                off += os.pwrite(fd, mv, off)
            os.close(fd)

    ths = [threading.Thread(target=work, args=(t,)) for t in range(threads)]
    t0 = time.perf_counter()
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    dt = time.perf_counter() - t0
    return threads * files_per * fsize / dt / 1e9


def main():
    d = sys.argv[1]
    threads = int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count()
    gib = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    per = int(gib * (1 << 30))
    os.makedirs(d, exist_ok=True)
    out = {"dir": d, "threads": threads, "bytes_per_thread": per}
    try:
        out["cmdline"] = open("/proc/cmdline").read().strip()
    except OSError:
        pass
    out["kernel"] = os.uname().release
    a = lambda t, f: os.path.join(d, f"a_{t}_{f}")  # noqa: E731
    b = lambda t, f: os.path.join(d, f"b_{t}_{f}")  # noqa: E731
    for rep in range(2):
        for name in os.listdir(d):
            os.unlink(os.path.join(d, name))
        out[f"fresh_GBps_{rep}"] = round(run(d, threads, per, "fresh", a), 2)
        out[f"overwrite_GBps_{rep}"] = round(run(d, threads, per, "overwrite", a), 2)
        files_per = max(1, per // (64 << 20))
        for t in range(threads):
            for f in range(files_per):
                os.rename(a(t, f), b(t, f))
        out[f"renamed_overwrite_GBps_{rep}"] = round(run(d, threads, per, "overwrite", b), 2)
    for name in os.listdir(d):
        os.unlink(os.path.join(d, name))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
