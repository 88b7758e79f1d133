#!/bin/bash
# full-size parity test + default bench (with restore verification) on 1 GPU
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_fullsize_gpu.py tests/test_memory_gpu.py -m gpu -x -q > gpurun_out/f_tests.log 2>&1; tail -3 gpurun_out/f_tests.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; tail -3 gpurun_out/f_bench.err
python -c "
import json
d=json.loads([l for l in open('gpurun_out/f_bench.json') if l.startswith('{')][-1])
print(d['value'], d['save_GBps'], d['restore_GBps'], d['restore_verified'], d['io_roofline']['save_frac'], d['io_roofline']['restore_frac'])"
