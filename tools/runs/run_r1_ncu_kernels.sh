#!/bin/bash
# ncu full sets of the current kernels: replica-parallel strided pack, reshard unpack, fused cast
cd "$(dirname "$0")/../.."
for c in rp_pack reshard_unpack; do
  K="python tools/kernel_bench.py --case $c --layers 8 --reps 3"
  $K > gpurun_out/nk_$c.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/nk_prof_$c -f $K > gpurun_out/nk_ncu_$c.log 2>&1
  echo "$c ncu rc=$?"; cat gpurun_out/nk_$c.log
done
C="python tools/cast_bench.py --layers 32"
$C > gpurun_out/nk_cast.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:box_cast -s 3 -c 1 -o gpurun_out/nk_prof_cast -f $C > gpurun_out/nk_ncu_cast.log 2>&1
echo "cast ncu rc=$?"; cat gpurun_out/nk_cast.log
