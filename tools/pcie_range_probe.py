"""PCIe evidence for the copy-engine legs of the engine: one pinned D2H and one pinned H2D
of 1 GiB, each inside its own cudaProfilerStart/Stop range, so that

    ncu --replay-mode range --profile-from-start off \
        --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum \
        python tools/pcie_range_probe.py

reports the PCIe bytes and the device time of exactly those transfers.  Without ncu it
prints the same transfers timed with CUDA events (GB/s)."""

import json
import time

import torch

N = 1 << 30


def main():
    dev = torch.empty(N, dtype=torch.uint8, device="cuda")
    host = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    dev.fill_(7)
    s = torch.cuda.current_stream()
    out = {}
    for name, fn in (("d2h", lambda: host.copy_(dev, non_blocking=True)),
                     ("h2d", lambda: dev.copy_(host, non_blocking=True))):
        fn()  # warm
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.profiler.start()
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.profiler.stop()
        torch.cuda.synchronize()
        out[name + "_GBps"] = round(N / (a.elapsed_time(b) / 1e3) / 1e9, 2)
        time.sleep(0.1)
    out["bytes"] = N
    print(json.dumps(out))


if __name__ == "__main__":
    main()
