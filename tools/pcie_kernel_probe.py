"""Is SM-driven PCIe (box-copy kernel reading/writing pinned host memory) as fast as the
copy engine?  Decides whether pack+D2H / H2D+unpack can be one fused kernel."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2605_23066_b200 import native  # noqa: E402


def timeit(fn, reps=5):
    s = torch.cuda.current_stream()
    for _ in range(2):
        fn(s)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn(s)
        b.record(s)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


for nbytes in (8 << 20, 64 << 20, 1 << 30):
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    host = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    n = nbytes // 16
    def ktab(src, dst):
        return native.copy_table([src], [(n,)], [(0,)], [dst], [(n,)], [(0,)], [(n,)], [16])
    d2h_tab = ktab(dev.data_ptr(), host.data_ptr())
    h2d_tab = ktab(host.data_ptr(), dev.data_ptr())
    res = {"bytes": nbytes}
    res["ce_d2h"] = nbytes / timeit(lambda s: host.copy_(dev, non_blocking=True)) / 1e6
    res["ce_h2d"] = nbytes / timeit(lambda s: dev.copy_(host, non_blocking=True)) / 1e6
    res["kernel_d2h"] = nbytes / timeit(lambda s: native.copy_boxes(0, d2h_tab, s.cuda_stream)) / 1e6
    res["kernel_h2d"] = nbytes / timeit(lambda s: native.copy_boxes(0, h2d_tab, s.cuda_stream)) / 1e6
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}), flush=True)
