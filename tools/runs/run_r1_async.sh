#!/bin/bash
# Async-step bench (live kernel timing) + ncu launch list / DRAM traffic of the same command.
cd "$(dirname "$0")/../.."
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q > gpurun_out/a_ktests.log 2>&1; tail -2 gpurun_out/a_ktests.log
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; tail -c 1500 gpurun_out/a_bench.json; tail -3 gpurun_out/a_bench.err
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none"
# pass-count check at 8 layers first: the full-size capture must be single-pass (no replay memory save)
timeout 600 ncu $M -c 20000 --csv --log-file gpurun_out/a_launches_8l.csv python bench.py --layers 8 --steps 1 --no-e2e --no-cpu-baseline --dir /dev/shm/tvncu > gpurun_out/a_ncu_8l.log 2>&1
grep -o "box_copy_kernel.*pass" gpurun_out/a_ncu_8l.log | sort | uniq -c | head
if grep -q "box_copy_kernel.* - 1 pass" gpurun_out/a_ncu_8l.log && ! grep -q "box_copy_kernel.* - [2-9] pass" gpurun_out/a_ncu_8l.log; then
  timeout 1500 ncu $M -c 50000 --csv --log-file gpurun_out/a_launches_full.csv python bench.py > gpurun_out/a_ncu_full.log 2>&1
  echo "full ncu rc=$?"; tail -c 300 gpurun_out/a_ncu_full.log
fi
