set -x
CUDA_VISIBLE_DEVICES=0 timeout 1500 python bench.py --steps 10 > gpurun_out/r2_v4b_n1.json 2> gpurun_out/r2_v4b_n1.err; echo n1 rc=$?
timeout 1500 python bench.py --gpus 2 --steps 10 > gpurun_out/r2_v4b_n2.json 2> gpurun_out/r2_v4b_n2.err; echo n2 rc=$?
timeout 1500 python bench.py --gpus 4 --steps 10 > gpurun_out/r2_v4b_n4.json 2> gpurun_out/r2_v4b_n4.err; echo n4 rc=$?
timeout 1500 python bench.py --gpus 4 --config c3 --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e > gpurun_out/r2_v4b_c3.json 2> gpurun_out/r2_v4b_c3.err; echo c3 rc=$?
timeout 1500 python bench.py --gpus 4 --config c4 --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e > gpurun_out/r2_v4b_c4.json 2> gpurun_out/r2_v4b_c4.err; echo c4 rc=$?
