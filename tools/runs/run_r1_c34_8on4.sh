#!/bin/bash
# BASELINE C3 (replica-parallel on a 2x4 mesh, 8 processes) and C4 (1x8 -> 2x4) with the
# driver's 8-rank torchrun shape on a 4-GPU box (2 ranks per GPU): robustness + parity
cd "$(dirname "$0")/../.."
for c in c3 c4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29645 \
    bench.py --gpus 8 --config $c --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/b8_$c.json 2> gpurun_out/b8_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/b8_$c.err | cut -c1-300
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/b8_$c.json') if l.startswith('{')][-1])
print(d['config']['workload'][:90], d['value'], d['save_GBps'], d['restore_GBps'], d['restore_verified']['mismatched_boxes'], d['restore_verified']['bytes_compared'], json.dumps(d['reshard_exchange'])[:80])"
done
