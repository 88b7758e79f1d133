#!/bin/bash
# Design probe: storage/PCIe options on the GPU box (results -> gpurun_out/io_probe.log)
cd "$(dirname "$0")/../.."
./tools/io_probe mem
for T in 8 16 32; do ./tools/io_probe /dev/shm 8 $T 256 32; ./tools/io_probe /dev/shm 8 $T 256 32; done
FALLOC=1 ./tools/io_probe /dev/shm 8 16 256 32
./tools/io_probe /dev/shm 8 16 64 4
./tools/io_probe /dev/shm 16 16 1024 64
