#!/bin/bash
cd "$(dirname "$0")/.."
timeout 600 python -m pytest tests/test_cast.py -m gpu -x -q > gpurun_out/cv_tests.log 2>&1; tail -2 gpurun_out/cv_tests.log
for L in 32; do
  echo "== layers $L default"; python tools/cast_bench.py --layers $L 2>&1 | tail -2
  for v in f g h i; do echo "== layers $L variant $v"; python tools/cast_bench.py --layers $L --lib tools/variants/libtvgpu_$v.so 2>&1 | tail -1; done
done
