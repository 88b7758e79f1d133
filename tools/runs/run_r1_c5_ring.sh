#!/bin/bash
# 1 GPU: small-ring engine sweep (DDIO-sized rings) + C5 Checkpointer every step x100.
cd "$(dirname "$0")/../.."
timeout 900 python tools/engine_sweep.py --layers 8 --reps 2 --settings 0.25:32,0.5:16,0.5:32,1:16,1:32,2:32,0.25:64 > gpurun_out/ring_sweep.jsonl 2> gpurun_out/ring_sweep.err
cat gpurun_out/ring_sweep.jsonl
timeout 900 python bench.py --config c5 --layers 8 --steps 100 --train-ms 1500 > gpurun_out/c5_100.json 2> gpurun_out/c5_100.err
tail -c 900 gpurun_out/c5_100.json
