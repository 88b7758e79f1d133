#!/bin/bash
# storage threads per rank under torchrun (huge tmpfs): default (cores-N)/N vs cores/N
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
C=$(nproc)
for t in default 12 default 12 default 10; do
  if [ "$t" = default ]; then E=""; else E="TVGPU_SLOTS=$t"; fi
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29627 bench.py --gpus $N --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/slc_$t.json 2>gpurun_out/slc_$t.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/slc_$t.json') if l.startswith('{')][-1])
r=d['io_roofline']; e=d['engine_rank0']
print('slots=$t', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], r['storage_write_GBps'], 'save_io', e['save']['thread_io_s'], 'load_io', e['load']['thread_io_s'])" >> gpurun_out/slc.txt 2>&1
  tail -1 gpurun_out/slc.txt
done
