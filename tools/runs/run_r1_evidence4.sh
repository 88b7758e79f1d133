#!/bin/bash
# 4-GPU evidence: torchrun parity tests, C3 replica-parallel and C4 reshard benches (threads
# runtime, NVLink fan-out), the fan-out kernel alone + its ncu NVLink / DRAM counters.
cd "$(dirname "$0")/../.."
N=$(python -c "import torch;print(torch.cuda.device_count())")
timeout 900 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/e4_dist_tests.log 2>&1; tail -1 gpurun_out/e4_dist_tests.log
for c in c4 c3; do
  timeout 1200 python bench.py --config $c --gpus $N --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/e4_$c.json 2> gpurun_out/e4_$c.err
  echo "$c rc=$?"; python -c "
import json,sys
d=json.loads([l for l in open('gpurun_out/e4_$c.json') if l.startswith('{')][-1])
print(d['value'], d['save_GBps'], d['restore_GBps'], json.dumps(d['io_roofline'])[:160]); print(json.dumps(d['reshard_exchange'])); print(json.dumps(d['roofline'])[:700])"
done
K="python tools/kernel_bench.py --case nvlink_fanout --layers 8 --reps 3"
$K > gpurun_out/e4_fanout.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum \
    --clock-control none -k regex:box_copy -c 8 --csv --log-file gpurun_out/e4_fanout_ncu.csv $K > gpurun_out/e4_fanout_ncu.log 2>&1
echo "fanout ncu rc=$?"; cat gpurun_out/e4_fanout.log; tail -12 gpurun_out/e4_fanout_ncu.csv | cut -c 1-40,300-
