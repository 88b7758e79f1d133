#!/bin/bash
# per_leaf vs aggregated layout (default bench otherwise), alternated x2
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for l in per_leaf aggregated per_leaf aggregated; do
  if [ "$N" = 1 ]; then
    timeout 900 python bench.py --layout $l --no-e2e --no-cpu-baseline > gpurun_out/ly${N}_$l.json 2>gpurun_out/ly${N}_$l.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29625 \
      bench.py --gpus $N --layout $l --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ly${N}_$l.json 2>gpurun_out/ly${N}_$l.err
  fi
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/ly${N}_$l.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('$l', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['restore_verified']['mismatched_boxes'])" >> gpurun_out/ly$N.txt 2>&1
  tail -1 gpurun_out/ly$N.txt
done
