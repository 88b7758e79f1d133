#!/bin/bash
# 8 ranks on a 4-GPU/32-core box: storage threads per rank 3 (default: (cores-8)/8) vs 4
cd "$(dirname "$0")/../.."
for t in default 4 default 4; do
  if [ "$t" = default ]; then E=""; else E="TVGPU_THREADS=$t"; fi
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 \
    --master-port 29647 bench.py --gpus 8 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/t8_$t.json 2>gpurun_out/t8_$t.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/t8_$t.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('threads=$t', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'])" >> gpurun_out/t8.txt 2>&1
  tail -1 gpurun_out/t8.txt
done
