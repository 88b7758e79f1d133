"""PCIe evidence for the copy-engine legs of the engine: one pinned D2H and one pinned H2D
of 1 GiB, each the only CUDA call inside its own cudaProfilerStart/Stop range, so that

    ncu --replay-mode range \
        --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum \
        python tools/pcie_range_probe.py

reports the PCIe bytes and the device time of exactly those transfers (range replay
records plain runtime memcpys; events or torch ops inside the range are not recordable,
so the ranges hold one cudaMemcpyAsync each and the timing events sit outside them).
Without ncu it prints the same transfers timed with CUDA events (GB/s)."""

import ctypes
import json
import os

N = 1 << 30


def cudart() -> ctypes.CDLL:
    for p in ("/usr/local/cuda/lib64/libcudart.so.12", "libcudart.so.12", "libcudart.so"):
        try:
            return ctypes.CDLL(p)
        except OSError:
            continue
    raise SystemExit("libcudart not found")


def main():
    rt = cudart()

    def ok(rc, what):
        if rc != 0:
            raise SystemExit(f"{what} failed: {rc}")

    P = ctypes.c_void_p
    dev, host, stream = P(), P(), P()
    ok(rt.cudaSetDevice(0), "cudaSetDevice")
    ok(rt.cudaMalloc(ctypes.byref(dev), ctypes.c_size_t(N)), "cudaMalloc")
    ok(rt.cudaHostAlloc(ctypes.byref(host), ctypes.c_size_t(N), 0), "cudaHostAlloc")
    ok(rt.cudaMemset(dev, 7, ctypes.c_size_t(N)), "cudaMemset")
    ok(rt.cudaStreamCreate(ctypes.byref(stream)), "cudaStreamCreate")
    ev = [P(), P()]
    for e in ev:
        ok(rt.cudaEventCreate(ctypes.byref(e)), "cudaEventCreate")
    out = {}
    for name, dst, src, kind in (("d2h", host, dev, 2), ("h2d", dev, host, 1)):
        ok(rt.cudaMemcpyAsync(dst, src, ctypes.c_size_t(N), kind, stream), "warm")
        ok(rt.cudaStreamSynchronize(stream), "sync")
        ok(rt.cudaEventRecord(ev[0], stream), "record")
        ok(rt.cudaProfilerStart(), "cudaProfilerStart")
        ok(rt.cudaMemcpyAsync(dst, src, ctypes.c_size_t(N), kind, stream), name)
        ok(rt.cudaProfilerStop(), "cudaProfilerStop")
        ok(rt.cudaEventRecord(ev[1], stream), "record")
        ok(rt.cudaStreamSynchronize(stream), "sync")
        ms = ctypes.c_float()
        ok(rt.cudaEventElapsedTime(ctypes.byref(ms), ev[0], ev[1]), "elapsed")
        out[name + "_GBps"] = round(N / (ms.value / 1e3) / 1e9, 2)
    out["bytes"] = N
    out["pid"] = os.getpid()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
