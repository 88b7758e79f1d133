#!/bin/bash
cd "$(dirname "$0")/../.."
cat /sys/devices/system/cpu/cpu0/cache/index3/size
mkdir -p /mnt/tvhuge && mount -t tmpfs -o size=150G,huge=always tmpfs /mnt/tvhuge
python tools/engine_sweep.py --layers 32 --reps 2 --dir /mnt/tvhuge/sweep --settings 0.25:64,0.5:64,1:32,1:64,2:16,2:32 > gpurun_out/sweep_huge2.log 2>&1; cat gpurun_out/sweep_huge2.log
umount -l /mnt/tvhuge
python tools/engine_sweep.py --layers 32 --reps 2 --settings 0.5:64,1:32,2:32 > gpurun_out/sweep_shm2.log 2>&1; cat gpurun_out/sweep_shm2.log
