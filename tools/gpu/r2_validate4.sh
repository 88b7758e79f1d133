set -x
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2_v4_gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2_v4_gputests.log
CUDA_VISIBLE_DEVICES=0 timeout 1500 python bench.py --steps 5 > gpurun_out/r2_v4_n1.json 2> gpurun_out/r2_v4_n1.err; echo n1 rc=$?
timeout 1500 python bench.py --gpus 4 --steps 5 > gpurun_out/r2_v4_n4.json 2> gpurun_out/r2_v4_n4.err; echo n4 rc=$?
timeout 1500 python bench.py --gpus 2 --steps 5 > gpurun_out/r2_v4_n2.json 2> gpurun_out/r2_v4_n2.err; echo n2 rc=$?
