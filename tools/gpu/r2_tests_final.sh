set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2_tf_build.log 2>&1; echo build rc=$?
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2_tf_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2_tf_gputests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_tf_smoke.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --config c5 --layers 8 --steps 30 > gpurun_out/r2_tf_c5.json 2> gpurun_out/r2_tf_c5.err; echo c5 rc=$?
timeout 900 python bench.py --config c1 --steps 10 > gpurun_out/r2_tf_c1.json 2> gpurun_out/r2_tf_c1.err; echo c1 rc=$?
