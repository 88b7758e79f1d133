#!/bin/bash
# /dev/shm vs a huge-page tmpfs mounted by bench.py (same engine, probe on the same mount)
cd "$(dirname "$0")/../.."
for st in shm hugetmpfs shm hugetmpfs; do
  timeout 900 python bench.py --storage $st --no-e2e --no-cpu-baseline > gpurun_out/st_$st.json 2>gpurun_out/st_$st.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/st_$st.json') if l.startswith('{')][-1])
r=d['io_roofline']
print('$st', d['value'], d['save_GBps'], d['restore_GBps'], r['bound'], r['storage_write_GBps'], r['storage_read_GBps'], r['save_frac'], r['restore_frac'], d['async_blocking_ms'])" >> gpurun_out/st.txt 2>&1
  tail -1 gpurun_out/st.txt
done
