import gc, os, sys, shutil, collections
sys.path.insert(0, os.getcwd())
import torch  # noqa: F401  (CUDA context before the package)
import bench
import paper_2605_23066_b200 as tv
base = "/dev/shm/tvcyc"; shutil.rmtree(base, ignore_errors=True)
backend = tv.FilesystemBackend(base)
rt = tv.SimulatedRuntime(1, backend, gpus=[0])
leaves = bench.llama_leaves(**dict(bench.LLAMA3_8B, layers=1))
mesh = tv.Mesh.create([("fsdp", 1)], process_count=1)
state, shardings = bench.build_state(tv, rt, mesh, leaves)
tv.save_checkpoint(rt, "a", state, shardings, tv.SaveOptions(sync=True)).wait()
gc.collect()
for what in ("save", "load"):
    gc.disable()
    gc.set_debug(gc.DEBUG_SAVEALL)
    if what == "save":
        h = tv.save_checkpoint(rt, "b", state, shardings, tv.SaveOptions(sync=False)); h.wait(); del h
    else:
        out = tv.load_checkpoint(rt, "a", None, tv.LoadOptions(), current_mesh=mesh); del out
    gc.collect()
    c = collections.Counter(type(o).__qualname__ for o in gc.garbage)
    print(what, len(gc.garbage), c.most_common(25))
    for o in gc.garbage:
        if type(o).__name__ in ("function",):
            print("  fn", o.__qualname__)
        if type(o).__name__ == "frame":
            print("  frame", o.f_code.co_name, o.f_code.co_filename.split("/")[-1], o.f_lineno)
        if type(o).__name__ in ("_RestoreJob", "SaveSession", "SaveHandle", "Thread"):
            print("  obj", type(o).__name__)
    gc.set_debug(0); gc.garbage.clear(); gc.enable()
