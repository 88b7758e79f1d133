set -x
timeout 1500 python bench.py --steps 10 > gpurun_out/r2_f1_n1.json 2> gpurun_out/r2_f1_n1.err; echo n1 rc=$?
timeout 900 python bench.py --impl reference --steps 4 --warmup 2 > gpurun_out/r2_f1_ref.json 2> gpurun_out/r2_f1_ref.err; echo ref rc=$?
timeout 600 python __graft_entry__.py smoke > gpurun_out/r2_f1_smoke.log 2>&1; echo smoke rc=$?
CMD="python bench.py --layers 4 --steps 2 --warmup 3 --c5-layers 0 --reshard-steps 1 --no-e2e --no-cpu-baseline --storage shm"
$CMD > gpurun_out/r2_ncu_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/r2_ncu_launches.csv $CMD > gpurun_out/r2_ncu_launch_run.log 2>&1; echo ncu1 rc=$?
$CMD > gpurun_out/r2_ncu_plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:box_copy -s 3 -c 1 -o gpurun_out/r2_ncu_snapshot $CMD > gpurun_out/r2_ncu_full_run.log 2>&1; echo ncu2 rc=$?
$CMD > gpurun_out/r2_ncu_plain3.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:box_copy -s 6 -c 2 -o gpurun_out/r2_ncu_unpack $CMD > gpurun_out/r2_ncu_full_run2.log 2>&1; echo ncu3 rc=$?
