set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_fl_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_fl_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_fl_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_fl_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fl_ref.json 2> gpurun_out/r2_fl_ref.err; echo ref rc=$?
t0=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fl_n1.json 2> gpurun_out/r2_fl_n1.err; echo n1 rc=$? wall=$(( $(date +%s) - t0 ))
CMD="python bench.py --layers 4 --steps 2 --warmup 3 --c5-layers 0 --reshard-steps 1 --no-e2e --no-cpu-baseline --c1-steps 0 --storage shm"
$CMD > gpurun_out/r2_fl_ncu_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_fl_ncu_launches.csv $CMD > gpurun_out/r2_fl_ncu_launch_run.log 2>&1; echo ncu1 rc=$?
$CMD > gpurun_out/r2_fl_ncu_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/r2_fl_ncu_snapshot $CMD > gpurun_out/r2_fl_ncu_full_run.log 2>&1; echo ncu2 rc=$?
