#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py --config c5 --layers 8 --steps 12 --train-ms 1000 > gpurun_out/cfg_c5c.log 2>&1; grep "^{" gpurun_out/cfg_c5c.log | cut -c1-150
python bench.py > gpurun_out/bench_full2.log 2>&1; grep "^{" gpurun_out/bench_full2.log | cut -c1-150
