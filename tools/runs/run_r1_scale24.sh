#!/bin/bash
# The driver's scaling shape on one 4-GPU box: default command at N=1, 2, 4 (torchrun for N>1).
cd "$(dirname "$0")/../.."
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/sc_1.json 2> gpurun_out/sc_1.err; echo "n1 rc=$?"
CUDA_VISIBLE_DEVICES=0,1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29641 bench.py --gpus 2 > gpurun_out/sc_2.json 2> gpurun_out/sc_2.err; echo "n2 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 \
  --master-port 29642 bench.py --gpus 4 > gpurun_out/sc_4.json 2> gpurun_out/sc_4.err; echo "n4 rc=$?"
for n in 1 2 4; do python -c "
import json
d=json.loads([l for l in open('gpurun_out/sc_$n.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('n=$n', d['value'], d['save_GBps'], d['restore_GBps'], r['bound'], r['save_frac'], r['restore_frac'], 'e2e', d['e2e']['value'], 'blk', d['async_blocking_ms'], 'ver', d['restore_verified']['mismatched_boxes'], d['per_process_last_step'])"; done
