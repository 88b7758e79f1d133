"""Fused-cast kernel microbenchmark: f32 master state -> bf16 (and i64 -> i32) converting
box copies of a Llama-3-8B FSDP-8 rank's f32 leaves, one launch; bytes = src + dst."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2605_23066_b200 import native  # noqa: E402
from tools.kernel_bench import shapes  # noqa: E402

import argparse  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--fsdp", type=int, default=8)
ap.add_argument("--lib", default=None, help="load this libtvgpu build instead (kernel variants)")
args = ap.parse_args()
if args.lib:
    from pathlib import Path

    native.LIB_PATH = Path(args.lib)
dev = torch.device("cuda", 0)
srcs, dsts = [], []
for shp in shapes(args.layers):
    src = torch.randn((shp[0] // args.fsdp,) + shp[1:], device=dev)
    srcs.append(src)
    dsts.append(torch.empty(src.shape, dtype=torch.bfloat16, device=dev))
flags = torch.zeros(1, dtype=torch.int32, device=dev)
n = len(srcs)
table = native.copy_table(
    [s.data_ptr() for s in srcs], [tuple(s.shape) for s in srcs], [(0,) * s.dim() for s in srcs],
    [d.data_ptr() for d in dsts], [tuple(d.shape) for d in dsts], [(0,) * d.dim() for d in dsts],
    [tuple(s.shape) for s in srcs], [4] * n, [native.DTYPE_CODE["f32"]] * n,
    [native.DTYPE_CODE["bf16"]] * n, [flags.data_ptr()] * n)
moved = sum(s.numel() * 6 for s in srcs)
from bench import time_launch  # noqa: E402

ms, host_ms = time_launch(lambda st: native.copy_boxes(0, table, st.cuda_stream), 0)
ok = all(torch.equal(d, s.to(torch.bfloat16)) for s, d in zip(srcs[:8], dsts[:8]))
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
# the same source bytes through the plain box copy (f32 -> f32), for comparison
cps = [torch.empty_like(s) for s in srcs]
ctab = native.copy_table(
    [s.data_ptr() for s in srcs], [tuple(s.shape) for s in srcs], [(0,) * s.dim() for s in srcs],
    [d.data_ptr() for d in cps], [tuple(d.shape) for d in cps], [(0,) * d.dim() for d in cps],
    [tuple(s.shape) for s in srcs], [4] * n)
cms, _ = time_launch(lambda st: native.copy_boxes(0, ctab, st.cuda_stream), 0)
cmoved = sum(s.numel() * 8 for s in srcs)
print(json.dumps({"case": "copy_f32_same_sources", "bytes": cmoved, "ms": round(cms, 3),
                  "achieved_GBps": round(cmoved / (cms / 1e3) / 1e9, 1)}))
print(json.dumps({"case": "cast_f32_to_bf16", "layers": args.layers, "copies": n, "bytes_src_plus_dst": moved, "ms": round(ms, 3), "host_enqueue_ms": round(host_ms, 3),
                  "achieved_GBps": round(moved / (ms / 1e3) / 1e9, 1), "peak_GBps": peak,
                  "frac": round(moved / (ms / 1e3) / 1e9 / peak, 4), "matches_torch_rne": ok,
                  "flags": int(flags.item())}))
