#!/bin/bash
# A/B on one box: sync-step vs async-step bench (C2 full), twice each, alternating.
cd "$(dirname "$0")/../.."
for m in sync async sync async; do
  timeout 900 python bench.py --save-mode $m --no-e2e --no-cpu-baseline > gpurun_out/ab_$m.json 2>gpurun_out/ab_$m.err
  python -c "
import json
d=json.loads([l for l in open('gpurun_out/ab_$m.json') if l.startswith('{')][-1])
e=d['engine_rank0']['save']
print('$m', d['value'], d['save_GBps'], d['restore_GBps'], d['io_roofline']['storage_write_GBps'], 'io_s', e['thread_io_s'], 'wall', e['wall_s'], 'sync_save_ms', d['sync_save_ms'], 'block', d['async_blocking_ms'])" >> gpurun_out/ab.txt
  tail -1 gpurun_out/ab.txt
done
P="python tools/pcie_range_probe.py"
$P > gpurun_out/ab_pcie.log 2>&1 && \
  ncu --replay-mode range --metrics pcie__read_bytes.sum,pcie__write_bytes.sum,gpu__time_duration.sum \
    --csv --log-file gpurun_out/ab_pcie_ncu.csv $P > gpurun_out/ab_pcie_ncu.log 2>&1
echo "pcie ncu rc=$?"; cat gpurun_out/ab_pcie.log; tail -8 gpurun_out/ab_pcie_ncu.csv; tail -5 gpurun_out/ab_pcie_ncu.log
