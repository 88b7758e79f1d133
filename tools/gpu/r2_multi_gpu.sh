set -x
nvidia-smi -L; nproc; free -g | head -2
timeout 600 python -m pytest tests/test_distributed.py -q -m gpu > gpurun_out/r2_mg_dist.log 2>&1; echo dist rc=$?
for N in 2 4; do
  timeout 1500 python bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r2_mg_c2_n$N.json 2> gpurun_out/r2_mg_c2_n$N.err; echo c2 n$N rc=$?
done
timeout 1500 python bench.py --gpus 4 --config c3 --steps 5 --warmup 3 --c5-layers 0 --reshard-steps 0 > gpurun_out/r2_mg_c3_n4.json 2> gpurun_out/r2_mg_c3_n4.err; echo c3 rc=$?
timeout 1500 python bench.py --gpus 4 --config c4 --steps 5 --warmup 3 --c5-layers 0 --reshard-steps 0 > gpurun_out/r2_mg_c4_n4.json 2> gpurun_out/r2_mg_c4_n4.err; echo c4 rc=$?
timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 8 --config c4 --restore-gpus 4 --steps 3 --warmup 2 --c5-layers 0 --reshard-steps 0 --no-e2e > gpurun_out/r2_mg_c4_8to4.json 2> gpurun_out/r2_mg_c4_8to4.err; echo c4_8to4 rc=$?
