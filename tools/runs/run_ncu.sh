#!/bin/bash
# ncu evidence (1 GPU): launch list of a (reduced) bench command, full sets of the kernels.
cd "$(dirname "$0")/../.."
B="python bench.py --layers 2 --steps 1 --warmup 3 --no-cpu-baseline --e2e-layers 1 --e2e-steps 1 --dir /dev/shm/tvncu"
$B > gpurun_out/ncu_bench_plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
tail -2 gpurun_out/ncu_launch.log
K="python tools/kernel_bench.py --case snapshot --layers 8 --reps 3"
$K > gpurun_out/kb_snap.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/prof_snapshot -f $K > gpurun_out/ncu_snap.log 2>&1
tail -1 gpurun_out/ncu_snap.log
C="python tools/cast_bench.py"
$C > gpurun_out/cast_plain.log 2>&1 && cat gpurun_out/cast_plain.log && \
  ncu --set full --clock-control none --import-source on -k regex:box_cast -s 2 -c 1 -o gpurun_out/prof_cast -f $C > gpurun_out/ncu_cast.log 2>&1
tail -1 gpurun_out/ncu_cast.log
