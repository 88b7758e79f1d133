#!/bin/bash
# What the driver runs at round end, 1 GPU: reference arm, gpu tests, smoke, default bench.
cd "$(dirname "$0")/../.."
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"; cut -c1-200 gpurun_out/fin_ref.json
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_gpu_tests.log 2>&1; tail -1 gpurun_out/fin_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; tail -1 gpurun_out/fin_smoke.log
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/fin_bench.json') if l.startswith('{')][-1])
r=d['io_roofline']
print(d['value'], d['save_GBps'], d['restore_GBps'], r['bound'], r['save_frac'], r['restore_frac'], d['async_blocking_ms'], d['sync_save_ms'])
print('e2e', json.dumps(d['e2e'])[:120]); print('cpu', json.dumps(d.get('cpu_baseline'))[:200]); print('roof', json.dumps(d['roofline'])[:300]); print('verified', d['restore_verified']['mismatched_boxes'], d['restore_verified']['bytes_compared']); print(d['config']['storage'])"
