set -x
timeout 900 python -m pytest tests/test_recycle_gpu.py tests/test_snapshot_gpu.py tests/test_distributed.py -q -x > gpurun_out/r2_f1b_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_f1b_tests.log
t0=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_f1b_n1.json 2> gpurun_out/r2_f1b_n1.err; echo n1 rc=$? wall=$(( $(date +%s) - t0 ))
