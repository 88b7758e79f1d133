#!/bin/bash
# Multi-GPU checks on a gpurun --gpus N box: topology probe, torchrun parity test, bench at N.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
{ nproc; free -g; df -h /dev/shm; nvidia-smi topo -m; } > gpurun_out/mg_probe.log 2>&1
timeout 600 python -m pytest tests/test_distributed.py -x -q > gpurun_out/mg_dist_tests.log 2>&1
tail -2 gpurun_out/mg_dist_tests.log
LAYERS=${LAYERS:-32}
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 \
  bench.py --gpus $N --layers $LAYERS ${BENCH_ARGS} > gpurun_out/mg_bench_$N.log 2>&1
tail -1 gpurun_out/mg_bench_$N.log | cut -c1-400
