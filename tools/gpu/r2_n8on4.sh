set -x
timeout 2400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 8 --steps 3 --warmup 5 > gpurun_out/r2_n8_on4.json 2> gpurun_out/r2_n8_on4.err; echo n8on4 rc=$?
