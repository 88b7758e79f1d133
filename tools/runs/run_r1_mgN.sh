#!/bin/bash
# Default bench under torchrun on all visible GPUs (the driver's scaling command) + dist tests
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 600 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/mg${N}_dist.log 2>&1; tail -1 gpurun_out/mg${N}_dist.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29613 \
  bench.py --gpus $N > gpurun_out/mg${N}_bench.json 2> gpurun_out/mg${N}_bench.err
echo "bench rc=$?"; tail -3 gpurun_out/mg${N}_bench.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/mg${N}_bench.json') if l.startswith('{')][-1])
print(d['value'], d['save_GBps'], d['restore_GBps'], d['io_roofline']['save_frac'], d['io_roofline']['restore_frac'], d['async_blocking_ms'], d['sync_save_ms'])
print(json.dumps(d['e2e'])); print(json.dumps(d['restore_verified'])); print(json.dumps(d['roofline'])[:400]); print(json.dumps(d['phases_ms_rank0_last_step']))"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29614 \
  bench.py --gpus $N --impl reference > gpurun_out/mg${N}_ref.json 2> gpurun_out/mg${N}_ref.err; echo "ref rc=$?"; cat gpurun_out/mg${N}_ref.json | cut -c1-300
