"""Box-copy kernel microbenchmark (the pack / unpack / snapshot kernel of the data path).

    python tools/kernel_bench.py [--case snapshot|rp_pack|reshard_unpack|all] [--layers L] [--reps R]

Cases (Llama-3-8B shapes, one GPU):
  snapshot        every shard of an FSDP-8 rank's state (10 GB) -> one arena, contiguous boxes
  rp_pack         C3 replica-parallel save: each (rows/4, cols) shard's column half
                  (a strided 2-D box: run = cols/2 elements) packed chunk-major
  reshard_unpack  C4 restore scatter: row-block chunks into (replica x fsdp) target shards
Each case is ONE launch for the whole batch; time = CUDA events on the launching stream,
median of R after 3 warm-ups.  Algorithmic bytes = 2 x bytes moved (read + write).
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_23066_b200 import native  # noqa: E402

D, FFN, V, KV = 4096, 14336, 128256, 1024


def shapes(layers):
    out = [(V, D), (V, D), (D,)]
    for _ in range(layers):
        out += [(D, D), (KV, D), (KV, D), (D, D), (FFN, D), (FFN, D), (D, FFN), (D,), (D,)]
    return out


def table(pairs):
    """pairs: (src_tensor, src_off, dst_tensor, dst_off, ext)"""
    copies = native.copy_table(
        [s.data_ptr() for s, _, _, _, _ in pairs], [tuple(s.shape) for s, _, _, _, _ in pairs],
        [so for _, so, _, _, _ in pairs], [t.data_ptr() for _, _, t, _, _ in pairs],
        [tuple(t.shape) for _, _, t, _, _ in pairs], [to for _, _, _, to, _ in pairs],
        [e for _, _, _, _, e in pairs], [s.element_size() for s, _, _, _, _ in pairs],
    )
    moved = sum(int(np.prod(e)) * s.element_size() for s, _, _, _, e in pairs)
    return copies, moved


def make_case(case, layers, fsdp=8):
    dev = torch.device("cuda", 0)
    pairs = []
    keep = []
    for tree, dt in (("params", torch.bfloat16), ("mu", torch.float32), ("nu", torch.float32)):
        for shp in shapes(layers):
            if case == "snapshot":
                src = torch.randn((shp[0] // fsdp,) + shp[1:], device=dev).to(dt)
                dst = torch.empty_like(src)
                pairs.append((src, (0,) * src.dim(), dst, (0,) * src.dim(), tuple(src.shape)))
                keep += [src, dst]
            elif case == "rp_pack":
                # 2x4 mesh, fsdp on dim 0: shard (rows/4, cols); replica r writes column half r
                rows = shp[0] // 4
                src = torch.randn((rows,) + shp[1:], device=dev).to(dt)
                if len(shp) == 1:
                    half = rows // 2
                    dst = torch.empty((half,), device=dev, dtype=dt)
                    pairs.append((src, (half,), dst, (0,), (half,)))
                else:
                    ext = (rows, shp[1] // 2) if shp[1] >= rows else (rows // 2, shp[1])
                    off = (0, shp[1] // 2) if shp[1] >= rows else (rows // 2, 0)
                    dst = torch.empty(ext, device=dev, dtype=dt)
                    pairs.append((src, off, dst, (0, 0), ext))
                keep += [src, dst]
            elif case == "reshard_unpack":
                # chunk = rows/8 block (from storage, contiguous) -> target shard rows/2 at an offset
                crow = shp[0] // 8
                chunk = torch.randn((crow,) + shp[1:], device=dev).to(dt)
                target = torch.empty((shp[0] // 2,) + shp[1:], device=dev, dtype=dt)
                for k in range(4):
                    pairs.append((chunk, (0,) * chunk.dim(), target, (k * crow,) + (0,) * (chunk.dim() - 1),
                                  tuple(chunk.shape)))
                keep += [chunk, target]
    copies, moved = table(pairs)
    return copies, moved, keep


def make_fanout(layers):
    """C4 restore fan-out over NVLink: row-block chunks landed on GPU 0 are written by a
    GPU-0 kernel straight into the replica's target shards on GPU 1 (P2P stores)."""
    from paper_2605_23066_b200 import native as nat

    nat.enable_peer_access([0, 1])
    pairs, keep = [], []
    for dt in (torch.bfloat16, torch.float32, torch.float32):
        for shp in shapes(layers):
            crow = shp[0] // 8
            chunk = torch.randn((crow,) + shp[1:], device="cuda:0").to(dt)
            target = torch.empty((shp[0] // 2,) + shp[1:], device="cuda:1", dtype=dt)
            for k in range(4):
                pairs.append((chunk, (0,) * chunk.dim(), target, (k * crow,) + (0,) * (chunk.dim() - 1),
                              tuple(chunk.shape)))
            keep += [chunk, target]
    copies, moved = table(pairs)
    return copies, moved, keep


def run(case, layers, reps, fsdp=8):
    if case == "nvlink_fanout":
        copies, moved, keep = make_fanout(layers)
    else:
        copies, moved, keep = make_case(case, layers, fsdp)
    from bench import time_launch

    ms, host_ms = time_launch(lambda st: native.copy_boxes(0, copies, st.cuda_stream), 0, reps=reps)
    torch.cuda.synchronize(0)
    if case == "nvlink_fanout":  # the peer stores really landed
        chunk, target = keep[0], keep[1]
        crow = chunk.shape[0]
        for k in range(4):
            assert torch.equal(target[k * crow:(k + 1) * crow].cpu(), chunk.cpu()), "fan-out mismatch"
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    achieved = 2 * moved / (ms / 1e3) / 1e9
    del keep
    torch.cuda.empty_cache()
    if case == "nvlink_fanout":  # bound: NVLink bytes leaving GPU 0 (770 GB/s measured peer copy)
        nv = moved / (ms / 1e3) / 1e9
        return {"case": case, "copies": len(copies), "bytes_moved": moved, "ms": round(ms, 3),
                "nvlink_GBps": round(nv, 1), "peak_GBps": 770.0, "frac": round(nv / 770.0, 4),
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s per direction"}
    return {"case": case, "copies": len(copies), "bytes_moved": moved, "ms": round(ms, 3),
            "host_enqueue_ms": round(host_ms, 3),
            "achieved_GBps": round(achieved, 1), "peak_GBps": peak, "frac": round(achieved / peak, 4)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="all")
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--reps", type=int, default=10)
    args = ap.parse_args()
    cases = ["snapshot", "rp_pack", "reshard_unpack"] if args.case == "all" else args.case.split(",")
    if args.case == "all" and torch.cuda.device_count() > 1:
        cases.append("nvlink_fanout")
    for c in cases:
        print(json.dumps(run(c, args.layers, args.reps)), flush=True)


if __name__ == "__main__":
    main()
