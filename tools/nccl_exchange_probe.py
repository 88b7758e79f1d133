"""Baseline for the restore's reshard exchange: NCCL moving the same bytes the fan-out
kernel stores into peer HBM (tools/kernel_bench.py --case nvlink_fanout: 13.98 GB
GPU0 -> GPU1 in one launch).  Run under torchrun with 2 ranks:

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        tools/nccl_exchange_probe.py [GB]

Prints one JSON line per case (rank 0): one-directional send/recv and a 2-rank
all_to_all_single, GB/s = bytes leaving one GPU / time (CUDA events, best of 5)."""

import json
import os
import sys

import torch
import torch.distributed as dist


def main():
    gb = float(sys.argv[1]) if len(sys.argv) > 1 else 13.98
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    n = int(gb * 1e9) // 16 * 16
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    buf.fill_(rank + 1)
    out = {}

    def timed(fn, reps=5):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        best = 1e30
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.barrier()
            a.record()
            fn()
            b.record()
            b.synchronize()
            best = min(best, a.elapsed_time(b))
        return best

    def send_recv():
        if rank == 0:
            dist.send(buf, 1)
        else:
            dist.recv(buf, 0)

    ms = timed(send_recv)
    out["nccl_send_recv_one_direction"] = {"bytes": n, "ms": round(ms, 3), "GBps": round(n / ms / 1e6, 1)}
    dst = torch.empty_like(buf)
    ms = timed(lambda: dist.all_to_all_single(dst, buf))
    half = n // 2  # each rank sends half of its buffer to the peer
    out["nccl_all_to_all_2rank"] = {"bytes_sent_per_gpu": half, "ms": round(ms, 3),
                                    "GBps_per_direction": round(half / ms / 1e6, 1)}
    if rank == 0:
        print(json.dumps({"case": "nccl_exchange_baseline", **out,
                          "nccl": ".".join(map(str, torch.cuda.nccl.version()))}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
