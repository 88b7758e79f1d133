#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/cast_bench.py > gpurun_out/cast_bench.log 2>&1; cat gpurun_out/cast_bench.log
python tools/engine_sweep.py --layers 32 --reps 2 --settings 2:32:16,2:30:15,2:28:14,2:24:12 > gpurun_out/sweep_threads.log 2>&1; cat gpurun_out/sweep_threads.log
