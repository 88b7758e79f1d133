set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_f4w_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_f4w_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_f4w_gputests.log
t0=$(date +%s); timeout 1500 python bench.py --gpus 4 --steps 10 > gpurun_out/r2_f4w_n4.json 2> gpurun_out/r2_f4w_n4.err; echo n4 rc=$? wall=$(( $(date +%s) - t0 ))
t0=$(date +%s); timeout 1500 python bench.py --gpus 2 --steps 10 > gpurun_out/r2_f4w_n2.json 2> gpurun_out/r2_f4w_n2.err; echo n2 rc=$? wall=$(( $(date +%s) - t0 ))
timeout 1500 python bench.py --gpus 4 --config c4 --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e --c1-steps 0 > gpurun_out/r2_f4w_c4.json 2> gpurun_out/r2_f4w_c4.err; echo c4 rc=$?
t0=$(date +%s); timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29617 bench.py --gpus 8 --steps 3 --warmup 3 > gpurun_out/r2_f4w_n8on4.json 2> gpurun_out/r2_f4w_n8on4.err; echo n8on4 rc=$? wall=$(( $(date +%s) - t0 ))
