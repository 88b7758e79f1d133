#!/bin/bash
# 8 torchrun ranks on the visible GPUs (2 per GPU on a 4-GPU box): the one-process-per-GPU
# runtime at the driver's largest world size — coordination, Checkpointer loop, byte-exact
# save from 8 ranks, IPC read-once reshard restore, IPC-free same-sharding restore, cast.
cd "$(dirname "$0")/../.."
for mode in coord datapath; do
  rm -rf /tmp/w8_$mode; mkdir -p /tmp/w8_$mode
  OMP_NUM_THREADS=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29641 tests/dist_worker.py $mode /tmp/w8_$mode > gpurun_out/w8_$mode.log 2>&1
  echo "$mode rc=$? ok_count=$(grep -c ' ok$' gpurun_out/w8_$mode.log)"
  grep -E "Error|error|assert" gpurun_out/w8_$mode.log | head -5
done
