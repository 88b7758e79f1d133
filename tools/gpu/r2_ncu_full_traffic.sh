set -x
CMD="python bench.py --steps 1 --warmup 3 --c5-layers 0 --reshard-steps 0 --no-e2e --c1-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/r2_nft_plain.json 2> gpurun_out/r2_nft_plain.err && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:box_copy -c 2 --csv --log-file gpurun_out/r2_nft_ncu.csv $CMD > gpurun_out/r2_nft_ncu_run.log 2>&1; echo ncu rc=$?
