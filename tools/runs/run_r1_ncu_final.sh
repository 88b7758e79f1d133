#!/bin/bash
# ncu launch list (+ DRAM bytes) of the default command, 1 GPU, after it exits 0 without ncu
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/nf_gpu_tests.log 2>&1; tail -1 gpurun_out/nf_gpu_tests.log
python bench.py > gpurun_out/nf_bench.json 2> gpurun_out/nf_bench.err && \
  timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 100000 --csv --log-file gpurun_out/nf_launches.csv python bench.py > gpurun_out/nf_ncu.log 2>&1
echo "rc=$?"; tail -c 300 gpurun_out/nf_bench.json
