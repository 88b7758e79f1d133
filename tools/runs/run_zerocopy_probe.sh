#!/bin/bash
cd "$(dirname "$0")/../.."
nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o /tmp/zc tools/zerocopy_probe.cu -lpthread 2>/dev/null
/tmp/zc /dev/shm 8 256 64
/tmp/zc /dev/shm 16 64 256
mkdir -p /mnt/tvhuge && mount -t tmpfs -o size=150G,huge=always tmpfs /mnt/tvhuge
/tmp/zc /mnt/tvhuge 8 256 64
/tmp/zc /mnt/tvhuge 16 64 256
umount -l /mnt/tvhuge
