set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_fm_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_fm_gputests.log
for pol in 1 0 1 0; do
TVGPU_GC_POLICY=$pol timeout 900 python bench.py --steps 5 --c5-layers 0 --no-e2e --c1-steps 0 --reshard-steps 3 --no-cpu-baseline >> gpurun_out/r2_fm_ab_n1.jsonl 2>> gpurun_out/r2_fm_ab_n1.err; echo ab pol=$pol rc=$?
done
t0=$(date +%s); timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_fm_n1.json 2> gpurun_out/r2_fm_n1.err; echo n1 rc=$? wall=$(( $(date +%s) - t0 ))
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_fm_smoke.log 2>&1; echo smoke rc=$?
