#!/bin/bash
# 4 GPUs: dist tests, the driver's default command under torchrun, torchrun C4 (IPC fan-out)
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 400 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/f4_dist.log 2>&1; tail -1 gpurun_out/f4_dist.log
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29621 \
  bench.py --gpus $N > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err; echo "bench rc=$?"
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29622 \
  bench.py --gpus $N --config c4 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/f4_c4.json 2> gpurun_out/f4_c4.err; echo "c4 rc=$?"
for f in f4_bench f4_c4; do python -c "
import json
d=json.loads([l for l in open('gpurun_out/$f.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('$f', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['async_blocking_ms'], d['sync_save_ms'], json.dumps(d.get('e2e'))[:60], d['restore_verified']['mismatched_boxes'], json.dumps(d['python_gc_rank0']))
print(json.dumps(d['phases_ms_rank0_last_step']))"; done
