#!/bin/bash
# slot-ring sizing on a huge-page tmpfs (PCIe-bound there), full C2, 1 GPU
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/hs_gpu_tests.log 2>&1; tail -2 gpurun_out/hs_gpu_tests.log
M=/mnt/tvsweep_huge; mkdir -p $M
KB=$(awk '/MemTotal/{print int($2*0.8)}' /proc/meminfo)
mount -t tmpfs -o size=${KB}k,huge=always tmpfs $M || exit 3
timeout 1200 python tools/engine_sweep.py --layers 32 --reps 2 --dir $M/s --settings 2:32,4:32,8:16,8:32,4:64 > gpurun_out/huge_sweep.jsonl 2> gpurun_out/huge_sweep.err
cat gpurun_out/huge_sweep.jsonl; tail -2 gpurun_out/huge_sweep.err
umount -l $M
