#!/bin/bash
# 1-GPU evidence: GPU suite, the default bench line, the ncu launch list + DRAM bytes of the
# SAME command, a full ncu set of the snapshot kernel, PCIe bytes of the copy-engine legs.
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/e_gpu_tests.log 2>&1; tail -2 gpurun_out/e_gpu_tests.log
python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err && \
  timeout 1800 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 100000 --csv --log-file gpurun_out/e_launches_full.csv python bench.py > gpurun_out/e_ncu_bench.log 2>&1
echo "bench+ncu rc=$?"; tail -c 400 gpurun_out/e_bench.json
K="python tools/kernel_bench.py --case snapshot --layers 8 --reps 3"
$K > gpurun_out/e_kb_snap.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/e_prof_snapshot -f $K > gpurun_out/e_ncu_snap.log 2>&1
echo "snap ncu rc=$?"; cat gpurun_out/e_kb_snap.log
P="python tools/pcie_range_probe.py"
$P > gpurun_out/e_pcie.log 2>&1 && \
  ncu --replay-mode range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum \
    --csv --log-file gpurun_out/e_pcie_ncu.csv $P > gpurun_out/e_pcie_ncu.log 2>&1
echo "pcie ncu rc=$?"; cat gpurun_out/e_pcie.log; cat gpurun_out/e_pcie_ncu.csv | tail -8
