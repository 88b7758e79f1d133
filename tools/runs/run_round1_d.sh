#!/bin/bash
cd "$(dirname "$0")/../.."
python bench.py --storage hugetmpfs --no-cpu-baseline --e2e-layers 1 > gpurun_out/bench_huge.log 2>&1; grep "^{" gpurun_out/bench_huge.log | cut -c1-100
python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log | cut -c1-300
