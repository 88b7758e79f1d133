#!/bin/bash
# Rank skew of the save's write phase under torchrun (per-process write_phase / engine_load),
# default storage threads vs oversubscribed (TVGPU_THREADS=10) — does a straggler tail exist?
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for t in default 10 default 10; do
  if [ "$t" = default ]; then E=""; else E="TVGPU_THREADS=$t"; fi
  env $E timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29633 bench.py --gpus $N --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/skew_$t.json 2>gpurun_out/skew_$t.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/skew_$t.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('threads=$t', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['restore_verified']['mismatched_boxes'], json.dumps(d['per_process_last_step']), d['phases_ms_rank0_last_step']['save']['barrier_written'])" >> gpurun_out/skew.txt 2>&1
  tail -1 gpurun_out/skew.txt
done
