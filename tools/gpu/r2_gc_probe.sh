set -x
TVGPU_GC_SOURCES=1 timeout 1200 python bench.py --gpus 4 --steps 10 --c5-layers 0 --no-e2e --c1-steps 0 --c3-steps 0 --reshard-steps 0 > gpurun_out/r2_gc_n4.json 2> gpurun_out/r2_gc_n4.err; echo n4 rc=$?
TVGPU_GC_SOURCES=1 timeout 1200 python bench.py --gpus 2 --steps 10 --c5-layers 0 --no-e2e --c1-steps 0 --c3-steps 0 --reshard-steps 0 > gpurun_out/r2_gc_n2.json 2> gpurun_out/r2_gc_n2.err; echo n2 rc=$?
