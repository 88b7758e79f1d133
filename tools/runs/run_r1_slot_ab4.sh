#!/bin/bash
# slot size A/B under torchrun on all visible GPUs (huge tmpfs): 1 / 2 / 4 MiB, x2
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for s in 1048576 2097152 4194304 1048576 2097152 4194304; do
  TVGPU_SLOT_BYTES=$s timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29617 bench.py --gpus $N --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/sl4_$s.json 2>gpurun_out/sl4_$s.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/sl4_$s.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('slot=$s', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], r['storage_write_GBps'], r['storage_read_GBps'])" >> gpurun_out/sl4.txt 2>&1
  tail -1 gpurun_out/sl4.txt
done
