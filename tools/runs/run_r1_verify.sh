#!/bin/bash
# Round-1 re-entry check of HEAD: full GPU suite, smoke, default bench line, cast bench.
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/v_gpu_tests.log 2>&1; tail -3 gpurun_out/v_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v_smoke.log 2>&1; tail -1 gpurun_out/v_smoke.log
timeout 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err; tail -c 600 gpurun_out/v_bench.json
timeout 300 python tools/cast_bench.py > gpurun_out/v_cast_bench.log 2>&1; tail -5 gpurun_out/v_cast_bench.log
