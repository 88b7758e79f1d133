#!/bin/bash
# Memoised restore planning under torchrun: C4 (reshard, CUDA-IPC consumers) and C3
# (replica-parallel), per-phase timelines; then the default C2 command at N GPUs.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for c in c4 c3 c2; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29616 \
    bench.py --gpus $N --config $c --steps 3 --warmup 3 > gpurun_out/pl${N}_$c.json 2> gpurun_out/pl${N}_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/pl${N}_$c.err | cut -c1-300
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/pl${N}_$c.json') if l.startswith('{')][-1])
r=d['io_roofline']
print(d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], json.dumps(d['restore_verified'])[:80])
print(json.dumps(d['phases_ms_rank0_last_step'])); print(d.get('python_gc_rank0')); print('e2e', json.dumps(d.get('e2e'))[:100])"
done
