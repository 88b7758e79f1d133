set -x
timeout 600 python tools/profile_host.py --c1 > gpurun_out/r2_prof_c1.txt 2>&1; echo prof rc=$?
