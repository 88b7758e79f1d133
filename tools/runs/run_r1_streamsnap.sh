#!/bin/bash
# stream-ordered snapshot: full GPU suite, default bench, C5 (8 layers x 40 steps)
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/ss_tests.log 2>&1; tail -1 gpurun_out/ss_tests.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/ss_bench.json 2> gpurun_out/ss_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/ss_bench.json') if l.startswith('{')][-1])
print(d['value'], d['save_GBps'], d['restore_GBps'], d['async_blocking_ms'], json.dumps(d['async_blocking_breakdown'])[:120], d['sync_save_ms'], d['async_blocking_frac_of_sync_save'], d['restore_verified']['mismatched_boxes'])"
timeout 900 python bench.py --config c5 --layers 8 --steps 40 --train-ms 1500 > gpurun_out/ss_c5.json 2> gpurun_out/ss_c5.err; echo "c5 rc=$?"
python -c "
import json
d=json.loads([l for l in open('gpurun_out/ss_c5.json') if l.startswith('{')][-1])
print({k: d[k] for k in ('value','blocking_host_ms_mean','snapshot_device_ms_mean','wait_on_previous_ms_mean','own_sync_phase_ms_mean','sync_save_ms','blocking_frac_of_sync_save')})"
