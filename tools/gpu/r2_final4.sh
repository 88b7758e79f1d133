set -x
timeout 1500 python -m pytest tests/test_baseline_sizes_gpu.py -q -x > gpurun_out/r2_f4_sizes.log 2>&1; echo sizes rc=$?; tail -2 gpurun_out/r2_f4_sizes.log
timeout 1500 python bench.py --gpus 4 --config c3 --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e --c1-steps 0 > gpurun_out/r2_f4_c3.json 2> gpurun_out/r2_f4_c3.err; echo c3 rc=$?
timeout 1500 python bench.py --gpus 2 --steps 10 > gpurun_out/r2_f4_n2.json 2> gpurun_out/r2_f4_n2.err; echo n2 rc=$?
timeout 1500 python bench.py --gpus 4 --steps 10 > gpurun_out/r2_f4_n4.json 2> gpurun_out/r2_f4_n4.err; echo n4 rc=$?
