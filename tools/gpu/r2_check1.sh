set -x
timeout 900 python -m pytest tests/test_recycle_gpu.py tests/test_gpu_parity.py tests/test_snapshot_gpu.py -q -x > gpurun_out/r2_c1_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_c1_tests.log
timeout 1500 python bench.py --steps 10 > gpurun_out/r2_c1_n1.json 2> gpurun_out/r2_c1_n1.err; echo n1 rc=$?
