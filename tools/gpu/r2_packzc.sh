set -x
timeout 900 python -m pytest tests/test_recycle_gpu.py tests/test_gpu_parity.py tests/test_random_parity_gpu.py -q -x > gpurun_out/r2_pz_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_pz_tests.log
