#!/bin/bash
# regression check: full GPU suite (2 GPUs) + the default bench line (GPU 0)
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c2_tests.log 2>&1; tail -1 gpurun_out/c2_tests.log
timeout 900 python bench.py > gpurun_out/c2_bench.json 2> gpurun_out/c2_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/c2_bench.json') if l.startswith('{')][-1])
r=d['io_roofline']
print(d['value'], d['save_GBps'], d['restore_GBps'], r['save_frac'], r['restore_frac'], d['async_blocking_ms'], d['e2e']['value'], d['cpu_baseline']['value'], d['restore_verified']['mismatched_boxes'], d['roofline']['frac'], d['roofline']['traffic'])"
