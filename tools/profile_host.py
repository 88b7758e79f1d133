"""Host-side (Python) cost of one save, one restore and one retire of the C2 tree (or,
with --c1, of the C1 tree: 4 x (4096,4096) f32 unsharded) at one GPU (the protocol around
the DMA): cProfile of each call, top functions by own time.

    python tools/profile_host.py [--layers 32] [--c1]
"""

from __future__ import annotations

import argparse
import cProfile
import io
import os
import pstats
import shutil
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--c1", action="store_true")
    args = ap.parse_args()
    import torch

    import bench
    import paper_2605_23066_b200 as tv
    from paper_2605_23066_b200.training_manager import delete_checkpoint

    base = "/dev/shm/tv_profile_host"
    shutil.rmtree(base, ignore_errors=True)
    backend = tv.FilesystemBackend(base)
    rt = tv.SimulatedRuntime(1, backend, gpus=[0])
    mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
    if args.c1:
        backend.register_pool = True  # as the bench's C1 leg
        state = {"model": {f"a{i}": tv.DenseArray("f32", torch.randn((4096, 4096), device="cuda"))
                           for i in range(4)}}
        shardings, mesh = None, None
    else:
        leaves = bench.llama_leaves(**dict(bench.LLAMA3_8B, layers=args.layers))
        state, shardings = bench.build_state(tv, rt, mesh, leaves)
    torch.cuda.synchronize()
    for i in range(6):  # warm: recycle pool, registrations, plan caches
        tv.save_checkpoint(rt, f"w{i}", state, shardings, tv.SaveOptions(sync=False)).wait()
        out = tv.load_checkpoint(rt, f"w{i}", None, tv.LoadOptions(), current_mesh=mesh)
        del out
        delete_checkpoint(backend.store(), f"w{i}", recycle=True)
    for what in ("save", "restore", "retire"):
        pr = cProfile.Profile()
        t0 = time.perf_counter()
        pr.enable()
        if what == "save":
            tv.save_checkpoint(rt, "p", state, shardings, tv.SaveOptions(sync=False)).wait()
        elif what == "restore":
            out = tv.load_checkpoint(rt, "p", None, tv.LoadOptions(), current_mesh=mesh)
            torch.cuda.synchronize()
        else:
            delete_checkpoint(backend.store(), "p", recycle=True)
        pr.disable()
        wall = (time.perf_counter() - t0) * 1e3
        s = io.StringIO()
        pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
        print(f"==== {what}: {wall:.1f} ms wall")
        print(s.getvalue())
        if what == "restore":
            from paper_2605_23066_b200 import timeline

            print(timeline.LAST_RESTORE)
    shutil.rmtree(base, ignore_errors=True)


if __name__ == "__main__":
    main()
