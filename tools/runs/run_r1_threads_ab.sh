#!/bin/bash
# A/B of storage threads per engine: default (cores - 1) vs all cores, full C2, 1 GPU.
cd "$(dirname "$0")/../.."
C=$(nproc)
for t in default $C default $C; do
  if [ "$t" = default ]; then E=""; else E="TVGPU_THREADS=$t"; fi
  env $E timeout 900 python bench.py --no-e2e --no-cpu-baseline > gpurun_out/thr_$t.json 2>gpurun_out/thr_$t.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/thr_$t.json') if l.startswith('{')][-1])
e=d['engine_rank0']
print('$t', d['value'], d['save_GBps'], d['restore_GBps'], d['io_roofline']['storage_write_GBps'], d['io_roofline']['storage_read_GBps'], 'save_io', e['save']['thread_io_s'], 'load_io', e['load']['thread_io_s'])" >> gpurun_out/thr.txt
  tail -1 gpurun_out/thr.txt
done
