#!/bin/bash
# IPC mapping cache: dist tests (2 GPUs: repeated IPC restores, cast across processes),
# torchrun C4 and C3 on all visible GPUs
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 400 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/ic_dist.log 2>&1; tail -1 gpurun_out/ic_dist.log
for c in c4 c3; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29661 \
    bench.py --gpus $N --config $c --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ic_$c.json 2> gpurun_out/ic_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/ic_$c.err | cut -c1-200
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/ic_$c.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('$c', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['restore_verified']['mismatched_boxes'], json.dumps({k: v for k, v in d['phases_ms_rank0_last_step']['restore'].items() if 'ipc' in k or k == 'engine_load'}))"
done
