set -x
timeout 2400 python bench.py --gpus 4 --config c5 --layers 32 --steps 100 --train-ms 2500 > gpurun_out/r2_c5fl_n4.json 2> gpurun_out/r2_c5fl_n4.err; echo c5 rc=$?
