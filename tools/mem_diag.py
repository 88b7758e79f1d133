"""Device-memory lifetime check: allocated bytes after each async save + restore step
(must return to the state's bytes without a gc.collect())."""
import gc
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_23066_b200 as tv  # noqa: E402

base = "/dev/shm/tvmem"
shutil.rmtree(base, ignore_errors=True)
backend = tv.FilesystemBackend(base)
rt = tv.SimulatedRuntime(1, backend, gpus=[0])
leaves = bench.llama_leaves(**dict(bench.LLAMA3_8B, layers=int(sys.argv[1]) if len(sys.argv) > 1 else 4))
mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
state, shardings = bench.build_state(tv, rt, mesh, leaves)
torch.cuda.synchronize()
GiB = 1 << 30
print("state", torch.cuda.memory_allocated() / GiB, flush=True)
for i in range(3):
    for sync in (False, True):
        h = tv.save_checkpoint(rt, f"s{i}{int(sync)}", state, shardings, tv.SaveOptions(sync=sync))
        h.wait()
        a1 = torch.cuda.memory_allocated() / GiB
        del h
        a2 = torch.cuda.memory_allocated() / GiB
        out = tv.load_checkpoint(rt, f"s{i}{int(sync)}", None, tv.LoadOptions(), current_mesh=mesh)
        a3 = torch.cuda.memory_allocated() / GiB
        del out
        a4 = torch.cuda.memory_allocated() / GiB
        gc.collect()
        a5 = torch.cuda.memory_allocated() / GiB
        print(f"step {i} sync={sync}: after save {a1:.2f} / handle dropped {a2:.2f} / restored {a3:.2f} "
              f"/ out dropped {a4:.2f} / gc {a5:.2f}", flush=True)
