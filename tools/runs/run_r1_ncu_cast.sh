#!/bin/bash
# ncu full set of the final (per-dtype-pair) cast kernel
cd "$(dirname "$0")/../.."
C="python tools/cast_bench.py --layers 32"
$C > gpurun_out/nc_cast.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:box_cast -s 3 -c 1 -o gpurun_out/nc_prof_cast -f $C > gpurun_out/nc_ncu_cast.log 2>&1
echo "cast ncu rc=$?"; cat gpurun_out/nc_cast.log
