#!/bin/bash
# BASELINE config 5 at full size: Checkpointer(keep_last=3) async save every step x100 of the
# 80.3 GB C2 state, FSDP over all visible GPUs under torchrun, 2.5 s synthetic training step.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
df -h /dev/shm | tail -1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29623 \
  bench.py --gpus $N --config c5 --layers 32 --steps 100 --train-ms ${TRAIN_MS:-2500} > gpurun_out/c5f_$N.json 2> gpurun_out/c5f_$N.err
echo "c5 rc=$?"; tail -c 1200 gpurun_out/c5f_$N.json; tail -3 gpurun_out/c5f_$N.err
