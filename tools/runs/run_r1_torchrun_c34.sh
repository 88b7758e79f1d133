#!/bin/bash
# torchrun C3 (replica-parallel 2xN/2) and C4 (1xN -> 2xN/2, same process count) benches,
# plus compute-sanitizer memcheck of the kernel unit tests and the smoke (GPU 0).
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
for c in c3 c4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29615 \
    bench.py --gpus $N --config $c --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/tr${N}_$c.json 2> gpurun_out/tr${N}_$c.err
  echo "$c rc=$?"; tail -2 gpurun_out/tr${N}_$c.err | cut -c1-300
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/tr${N}_$c.json') if l.startswith('{')][-1])
print(d['value'], d['save_GBps'], d['restore_GBps'], d['io_roofline']['save_frac'], d['io_roofline']['restore_frac'], json.dumps(d['restore_verified'])[:80], json.dumps(d['reshard_exchange'])[:90])
print(json.dumps(d['roofline'])[:600])"
done
CUDA_VISIBLE_DEVICES=0 timeout 1200 compute-sanitizer --tool memcheck --leak-check no --error-exitcode 9 \
  python -m pytest tests/test_kernels_gpu.py tests/test_cast.py -m gpu -x -q > gpurun_out/tr_memcheck.log 2>&1
echo "memcheck rc=$?"; tail -5 gpurun_out/tr_memcheck.log
