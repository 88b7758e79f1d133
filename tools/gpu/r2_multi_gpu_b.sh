set -x
mkdir -p /mnt/h && mount -t tmpfs -o size=200g,huge=always tmpfs /mnt/h
for g in 0 1 2 3; do CUDA_VISIBLE_DEVICES=$g timeout 300 ./tools/mapped_dma_probe /mnt/h/g$g 16 1024 3 > gpurun_out/r2_mapped_probe_4gpu_$g.json 2>&1 & done; mkdir -p /mnt/h/g0 /mnt/h/g1 /mnt/h/g2 /mnt/h/g3; wait
for g in 0 1 2 3; do mkdir -p /mnt/h/g$g; done
for g in 0 1 2 3; do CUDA_VISIBLE_DEVICES=$g timeout 300 ./tools/mapped_dma_probe /mnt/h/g$g 16 1024 3 > gpurun_out/r2_mapped_probe_4gpu_$g.json 2>&1 & done; wait
umount /mnt/h
timeout 600 python -m pytest tests/test_distributed.py -q -m gpu > gpurun_out/r2_mg_dist.log 2>&1; echo dist rc=$?
for N in 2 4; do
  timeout 1500 python bench.py --gpus $N --steps 5 --warmup 3 > gpurun_out/r2_mg_c2_n$N.json 2> gpurun_out/r2_mg_c2_n$N.err; echo c2 n$N rc=$?
done
timeout 1500 python bench.py --gpus 4 --config c4 --steps 5 --warmup 3 --c5-layers 0 --reshard-steps 0 > gpurun_out/r2_mg_c4_n4.json 2> gpurun_out/r2_mg_c4_n4.err; echo c4 rc=$?
