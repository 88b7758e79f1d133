#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 400 python -m pytest tests/test_distributed.py -m gpu -x -q > gpurun_out/dd_tests.log 2>&1; tail -3 gpurun_out/dd_tests.log | cut -c1-600
