set -x
timeout 900 python tools/conformance.py --out gpurun_out/r2_conformance_final; echo conf rc=$?
for mode in torchrun threads torchrun threads; do
  timeout 1500 python bench.py --gpus 4 --runtime $mode --steps 5 --c5-layers 0 --reshard-steps 0 --no-e2e --c1-steps 0 >> gpurun_out/r2_ab_runtime_n4.jsonl 2>> gpurun_out/r2_ab_runtime_n4.err; echo $mode rc=$?
done
timeout 2400 python bench.py --gpus 4 --config c5 --layers 32 --steps 100 --train-ms 2500 > gpurun_out/r2_c5_full_n4.json 2> gpurun_out/r2_c5_full_n4.err; echo c5 rc=$?
