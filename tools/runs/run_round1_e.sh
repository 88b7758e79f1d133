#!/bin/bash
cd "$(dirname "$0")/../.."
mkdir -p /mnt/tvhuge && mount -t tmpfs -o size=150G,huge=always tmpfs /mnt/tvhuge
python tools/engine_sweep.py --layers 32 --reps 2 --dir /mnt/tvhuge/sweep --settings 2:32,2:96,8:32,8:64,16:32,32:16 > gpurun_out/sweep_huge.log 2>&1; cat gpurun_out/sweep_huge.log
umount -l /mnt/tvhuge
