set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_fw_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_fw_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_fw_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_fw_smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fw_ref.json 2> gpurun_out/r2_fw_ref.err; echo ref rc=$?
t0=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fw_n1.json 2> gpurun_out/r2_fw_n1.err; echo n1 rc=$? wall=$(( $(date +%s) - t0 ))
