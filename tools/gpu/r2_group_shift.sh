set -x
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_gpu_parity.py tests/test_random_parity_gpu.py tests/test_reshard_large_gpu.py -q -x > gpurun_out/r2_gs_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/r2_gs_tests.log
timeout 600 tools/tma2d_pack_probe > gpurun_out/r2_gs_new.jsonl 2> gpurun_out/r2_gs.err; echo new rc=$?
LD_LIBRARY_PATH=$PWD/tools/old_lib timeout 600 tools/tma2d_pack_probe > gpurun_out/r2_gs_old.jsonl 2>> gpurun_out/r2_gs.err; echo old rc=$?
timeout 600 tools/tma2d_pack_probe > gpurun_out/r2_gs_new2.jsonl 2>> gpurun_out/r2_gs.err; echo new2 rc=$?
LD_LIBRARY_PATH=$PWD/tools/old_lib timeout 600 tools/tma2d_pack_probe > gpurun_out/r2_gs_old2.jsonl 2>> gpurun_out/r2_gs.err; echo old2 rc=$?
