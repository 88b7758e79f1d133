#!/bin/bash
# Extra bench configurations on a 1-GPU box (results -> gpurun_out/cfg_*.log)
cd "$(dirname "$0")/../.."
python bench.py --config c1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_c1.log 2>&1; tail -1 gpurun_out/cfg_c1.log | cut -c1-200
python bench.py --config c5 --layers 8 --steps 20 --train-ms 1000 > gpurun_out/cfg_c5.log 2>&1; tail -1 gpurun_out/cfg_c5.log | cut -c1-300
python bench.py --config c3 --gpus 2 --layers 8 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/cfg_c3_emul.log 2>&1; tail -1 gpurun_out/cfg_c3_emul.log | cut -c1-200
