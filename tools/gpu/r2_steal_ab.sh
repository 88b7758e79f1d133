set -x
for st in 0 1; do
  TVGPU_SAVE_STEAL=$st timeout 1500 python bench.py --gpus 4 --steps 5 --warmup 3 --c5-layers 0 --reshard-steps 0 --no-e2e > gpurun_out/r2_steal${st}_n4.json 2> gpurun_out/r2_steal${st}_n4.err; echo n4 steal$st rc=$?
done
TVGPU_SAVE_STEAL=1 timeout 1500 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2_steal1_n2.json 2> gpurun_out/r2_steal1_n2.err; echo n2 rc=$?
for st in 0 1; do
  CUDA_VISIBLE_DEVICES=0 TVGPU_SAVE_STEAL=$st timeout 1500 python bench.py --steps 5 --warmup 3 --c5-layers 0 --reshard-steps 0 --no-e2e --no-cpu-baseline > gpurun_out/r2_steal${st}_n1.json 2> gpurun_out/r2_steal${st}_n1.err; echo n1 steal$st rc=$?
done
