#!/bin/bash
# Where the Python cyclic GC is triggered during the timed steps (allocation sites), 1 GPU.
cd "$(dirname "$0")/../.."
TVGPU_GC_SOURCES=1 timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/gcs.json 2> gpurun_out/gcs.err
echo "rc=$?"; tail -2 gpurun_out/gcs.err | cut -c1-300
python -c "
import json
d=json.loads([l for l in open('gpurun_out/gcs.json') if l.startswith('{')][-1])
g=d['python_gc_rank0']; print(g['ms_per_step'], g['collections'], g['gen2'])
for s in g['sources']: print(s)"
