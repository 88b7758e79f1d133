set -x
for i in 1 2; do
TVGPU_GC_SOURCES=1 timeout 900 python bench.py --config c5 --layers 8 --steps 30 > gpurun_out/r2_c5chk_$i.json 2> gpurun_out/r2_c5chk_$i.err; echo c5 $i rc=$?
done
