#!/bin/bash
# slot size A/B on the default bench (huge tmpfs, 1 GPU): 2 MiB (default) vs 4 MiB, x3
cd "$(dirname "$0")/../.."
for s in 2097152 4194304 2097152 4194304 2097152 4194304; do
  TVGPU_SLOT_BYTES=$s timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/sl_$s.json 2>gpurun_out/sl_$s.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/sl_$s.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('slot=$s', d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'])" >> gpurun_out/sl.txt 2>&1
  tail -1 gpurun_out/sl.txt
done
