set -x
for pol in 1 0 1 0; do
TVGPU_GC_POLICY=$pol TVGPU_GC_SOURCES=1 timeout 1200 python bench.py --gpus 4 --steps 10 --c5-layers 0 --no-e2e --c1-steps 0 --c3-steps 0 --reshard-steps 0 >> gpurun_out/r2_gcab_n4.jsonl 2>> gpurun_out/r2_gcab_n4.err; echo n4 pol=$pol rc=$?
done
timeout 900 python -m pytest tests/test_distributed.py tests/test_gpu_parity.py -q -x > gpurun_out/r2_gcab_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_gcab_tests.log
