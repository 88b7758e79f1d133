#!/bin/bash
# ncu evidence for the box-copy kernel + C5 timeline + engine sweep (1 GPU)
cd "$(dirname "$0")/../.."
python bench.py --config c5 --layers 8 --steps 12 --train-ms 1000 > gpurun_out/cfg_c5b.log 2>&1; grep "^{" gpurun_out/cfg_c5b.log | cut -c1-200
python tools/engine_sweep.py --layers 8 > gpurun_out/engine_sweep.log 2>&1; cat gpurun_out/engine_sweep.log
KB="python tools/kernel_bench.py --case rp_pack --layers 4 --reps 3"
$KB > gpurun_out/kb_plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/prof_rp_pack -f $KB > gpurun_out/ncu_full.log 2>&1
tail -3 gpurun_out/ncu_full.log
