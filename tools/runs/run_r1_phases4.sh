#!/bin/bash
# C2 under torchrun on all visible GPUs with per-phase timelines (host overhead vs engine).
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for cfg in "default:" "s512k32:TVGPU_SLOT_BYTES=524288 TVGPU_SLOTS=32"; do
  tag=${cfg%%:*}; envs=${cfg#*:}
  env $envs timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 29612 bench.py --gpus $N --steps 2 --warmup 2 --no-e2e --no-cpu-baseline ${BENCH_ARGS} \
    > gpurun_out/ph${N}_$tag.log 2>&1
  grep "^{" gpurun_out/ph${N}_$tag.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$tag', d['value'], d['save_GBps'], d['restore_GBps'], d['save_ms'], d['restore_ms'], json.dumps(d['io_roofline'])[:200])
print(json.dumps(d['phases_ms_rank0_last_step']))
print(json.dumps(d['engine_rank0']))"
done
