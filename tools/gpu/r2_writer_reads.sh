set -x
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_random_parity_gpu.py tests/test_reshard_large_gpu.py tests/test_distributed.py tests/test_baseline_sizes_gpu.py tests/test_acceptance_gpu.py -q -x > gpurun_out/r2_wr_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_wr_tests.log
for wr in 1 0; do
  TVGPU_WRITER_READS=$wr timeout 1500 python bench.py --gpus 4 --steps 5 --c5-layers 0 --no-e2e --c1-steps 0 > gpurun_out/r2_wr${wr}_n4.json 2> gpurun_out/r2_wr${wr}_n4.err; echo n4 wr$wr rc=$?
  TVGPU_WRITER_READS=$wr timeout 1500 python bench.py --gpus 4 --config c4 --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e --c1-steps 0 > gpurun_out/r2_wr${wr}_c4.json 2> gpurun_out/r2_wr${wr}_c4.err; echo c4 wr$wr rc=$?
done
