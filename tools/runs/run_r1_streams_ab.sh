#!/bin/bash
# DMA streams per device: parity under 4 streams, then bench A/B 1 / 2 / 4 (huge tmpfs, 1 GPU)
cd "$(dirname "$0")/../.."
TVGPU_DMA_STREAMS=4 timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ds_tests.log 2>&1; tail -2 gpurun_out/ds_tests.log
for n in 1 2 4 1 2 4; do
  TVGPU_DMA_STREAMS=$n timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/ds_$n.json 2>gpurun_out/ds_$n.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/ds_$n.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('streams=$n', d['value'], d['save_GBps'], d['restore_GBps'], r['bound'], r['save_peak_GBps'], r['restore_peak_GBps'], r['save_frac'], r['restore_frac'])" >> gpurun_out/ds.txt 2>&1
  tail -1 gpurun_out/ds.txt
done
