#!/bin/bash
# huge-page (THP) slot ring vs cudaHostAlloc slots, 1 GPU, default bench, x3 alternating
cd "$(dirname "$0")/../.."
TVGPU_HUGE_RING=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_random_parity_gpu.py -m gpu -x -q > gpurun_out/hr_tests.log 2>&1; tail -1 gpurun_out/hr_tests.log
for h in 0 1 0 1 0 1; do
  TVGPU_HUGE_RING=$h timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/hr_$h.json 2>gpurun_out/hr_$h.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/hr_$h.json') if l.startswith('{')][-1])
r=d['io_roofline']; c=r['contended']
print('huge=$h', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], 'contended d2h', c['d2h_GBps'], 'wait_dma', d['engine_rank0']['save']['thread_wait_dma_s'])" >> gpurun_out/hr.txt 2>&1
  tail -1 gpurun_out/hr.txt
done
