#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 900 python -m pytest tests/test_random_parity_gpu.py -m gpu -q > gpurun_out/rp_tests.log 2>&1; tail -15 gpurun_out/rp_tests.log | cut -c1-400
