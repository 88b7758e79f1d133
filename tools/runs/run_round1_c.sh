#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py --config c5 --layers 8 --steps 12 --train-ms 1000 > gpurun_out/cfg_c5c.log 2>&1; grep "^{" gpurun_out/cfg_c5c.log | cut -c1-150
python tools/engine_sweep.py --layers 32 --reps 2 > gpurun_out/engine_sweep32.log 2>&1; cat gpurun_out/engine_sweep32.log
