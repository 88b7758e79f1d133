set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_f4l_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_f4l_gputests.log
t0=$(date +%s); timeout 1500 python bench.py --gpus 4 --steps 10 > gpurun_out/r2_f4l_n4.json 2> gpurun_out/r2_f4l_n4.err; echo n4 rc=$? wall=$(( $(date +%s) - t0 ))
t0=$(date +%s); timeout 1500 python bench.py --gpus 2 --steps 10 > gpurun_out/r2_f4l_n2.json 2> gpurun_out/r2_f4l_n2.err; echo n2 rc=$? wall=$(( $(date +%s) - t0 ))
