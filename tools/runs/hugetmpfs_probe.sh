#!/bin/bash
# Does a huge-page tmpfs change the storage roofline? (design probe)
cd "$(dirname "$0")/../.."
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/io_probe tools/io_probe.cu -lpthread 2>/dev/null
mkdir -p /mnt/tvhuge && mount -t tmpfs -o size=120G,huge=always tmpfs /mnt/tvhuge && echo mounted-huge
cat /proc/mounts | grep tvhuge
for i in 1 2; do /tmp/io_probe /dev/shm 16 16 256 8; done
for i in 1 2; do /tmp/io_probe /mnt/tvhuge 16 16 256 8; done
grep -i huge /proc/meminfo
umount /mnt/tvhuge
