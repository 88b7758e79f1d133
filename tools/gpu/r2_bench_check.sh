set -x
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bc_n1.json 2> gpurun_out/r2_bc_n1.err; echo n1 rc=$?
