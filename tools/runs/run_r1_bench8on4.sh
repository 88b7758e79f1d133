#!/bin/bash
# the driver's N=8 command shape (torchrun, 8 ranks) on a 4-GPU box: robustness, not speed
cd "$(dirname "$0")/../.."
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29643 \
  bench.py --gpus 8 --steps 2 --warmup 3 > gpurun_out/b8_bench.json 2> gpurun_out/b8_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/b8_bench.err | cut -c1-300
python -c "
import json
d=json.loads([l for l in open('gpurun_out/b8_bench.json') if l.startswith('{')][-1])
r=d['io_roofline']
print(d['n_gpus'], d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['restore_verified'], json.dumps(d['e2e'])[:80], d['gpu_launches'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29644 \
  bench.py --gpus 8 --impl reference --steps 2 --warmup 1 > gpurun_out/b8_ref.json 2> gpurun_out/b8_ref.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/b8_ref.json
