#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 600 python -m pytest tests/test_cast.py tests/test_kernels_gpu.py tests/test_acceptance_gpu.py -m gpu -x -q > gpurun_out/cv3_tests.log 2>&1; tail -2 gpurun_out/cv3_tests.log
for L in 8 32; do python tools/cast_bench.py --layers $L 2>&1 | tail -2; done
