#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t2_tests.log 2>&1; tail -1 gpurun_out/t2_tests.log
