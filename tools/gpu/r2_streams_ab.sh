set -x
for s in 1 2 1 2; do
TVGPU_DMA_STREAMS=$s timeout 900 python bench.py --gpus 4 --steps 3 --warmup 3 --c5-layers 0 --no-e2e --c1-steps 0 --c3-steps 0 --reshard-steps 0 >> gpurun_out/r2_streams_n4.jsonl 2>> gpurun_out/r2_streams_n4.err; echo s=$s rc=$?
done
