"""cProfile of the blocking part of an async save of the C2 state on one GPU."""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_23066_b200 as tv  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
base = "/dev/shm/tvprof"
os.makedirs(base, exist_ok=True)
backend = tv.FilesystemBackend(base)
rt = tv.SimulatedRuntime(1, backend, gpus=[0])
dims = dict(bench.LLAMA3_8B, layers=layers)
leaves = bench.llama_leaves(**dims)
mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
state, shardings = bench.build_state(tv, rt, mesh, leaves)
torch.cuda.synchronize()
for i in range(2):
    t0 = time.perf_counter()
    h = tv.save_checkpoint(rt, f"p/warm{i}", state, shardings, tv.SaveOptions(sync=False))
    print("blocking ms", (time.perf_counter() - t0) * 1e3)
    h.wait()
    import shutil
    shutil.rmtree(os.path.join(base, "p"), ignore_errors=True)
prof = cProfile.Profile()
t0 = time.perf_counter()
prof.enable()
h = tv.save_checkpoint(rt, "p/prof", state, shardings, tv.SaveOptions(sync=False))
prof.disable()
print("profiled blocking ms", (time.perf_counter() - t0) * 1e3)
pstats.Stats(prof).sort_stats("cumulative").print_stats(40)
pstats.Stats(prof).sort_stats("tottime").print_stats(25)
h.wait()
import shutil
shutil.rmtree(base, ignore_errors=True)
