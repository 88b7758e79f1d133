#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
python tools/kernel_bench.py > gpurun_out/kernel_bench2.log 2>&1; cat gpurun_out/kernel_bench2.log
python tools/cast_bench.py > gpurun_out/cast_bench.log 2>&1; cat gpurun_out/cast_bench.log
python bench.py > gpurun_out/bench_full4.log 2>&1; grep "^{" gpurun_out/bench_full4.log | cut -c1-100
