#!/bin/bash
# NUMA placement path under torchrun: default (auto: no-op on a single-node host) vs
# TVGPU_NUMA=force (binds each rank's engine to its GPU's local_cpulist even on one node).
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
ls /sys/devices/system/node/ | grep node; cat /sys/devices/system/node/node*/cpulist
for t in force default; do
  if [ "$t" = default ]; then E=""; else E="TVGPU_NUMA=$t"; fi
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29631 bench.py --gpus $N --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/numa_$t.json 2>gpurun_out/numa_$t.err
  echo "$t rc=$?"; tail -1 gpurun_out/numa_$t.err | cut -c1-300
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/numa_$t.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('$t', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['restore_verified']['mismatched_boxes'], json.dumps(d['numa_rank0'])[:200])"
done
