#!/bin/bash
# Reshard exchange: the fan-out kernel (P2P stores, one launch) vs NCCL on the same bytes
cd "$(dirname "$0")/../.."
timeout 300 python tools/kernel_bench.py --case nvlink_fanout --layers 8 --reps 5 > gpurun_out/nx_fanout.log 2>&1; cat gpurun_out/nx_fanout.log
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 \
  tools/nccl_exchange_probe.py 13.98 > gpurun_out/nx_nccl.log 2>&1; grep "^{" gpurun_out/nx_nccl.log || tail -5 gpurun_out/nx_nccl.log
