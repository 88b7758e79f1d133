#!/bin/bash
# Multi-GPU round: N = visible GPUs.  Topology, torchrun parity, C2 (torchrun), C3 + C4
# (threads runtime, NVLink P2P fan-out), NVLink fan-out kernel.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
{ nproc; free -g; df -h /dev/shm; nvidia-smi topo -m; cat /sys/devices/system/cpu/cpu0/cache/index3/size; } > gpurun_out/mg${N}_probe.log 2>&1
timeout 600 python -m pytest tests/test_distributed.py -x -q > gpurun_out/mg${N}_dist_tests.log 2>&1; tail -1 gpurun_out/mg${N}_dist_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29600 \
  bench.py --gpus $N ${C2ARGS} > gpurun_out/mg${N}_c2.log 2>&1; grep "^{" gpurun_out/mg${N}_c2.log | cut -c1-120
timeout 1200 python bench.py --config c3 --gpus $N --no-cpu-baseline --no-e2e ${C34ARGS} > gpurun_out/mg${N}_c3.log 2>&1; grep "^{" gpurun_out/mg${N}_c3.log | cut -c1-120
timeout 1200 python bench.py --config c4 --gpus $N --no-cpu-baseline --no-e2e ${C34ARGS} > gpurun_out/mg${N}_c4.log 2>&1; grep "^{" gpurun_out/mg${N}_c4.log | cut -c1-120
python tools/kernel_bench.py --case nvlink_fanout --layers 8 > gpurun_out/mg${N}_nvlink.log 2>&1; cat gpurun_out/mg${N}_nvlink.log
