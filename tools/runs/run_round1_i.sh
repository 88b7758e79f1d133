#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests/test_cast.py tests/test_kernels_gpu.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/gpu_tests_cast.log 2>&1; tail -2 gpurun_out/gpu_tests_cast.log
C="python tools/cast_bench.py"
$C > gpurun_out/cast_bench.log 2>&1 && cat gpurun_out/cast_bench.log && \
  ncu --set full --clock-control none --import-source on -k regex:box_cast -s 2 -c 1 -o gpurun_out/prof_cast2 -f $C > gpurun_out/ncu_cast2.log 2>&1
tail -1 gpurun_out/ncu_cast2.log
