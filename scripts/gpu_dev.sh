#!/bin/bash
# Development GPU session (round 2): new parity tests, kernel variants, full GPU suite.
# Usage: bash scripts/gpu_dev.sh <tag>
TAG=${1:-dev}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests/test_gpu_exponents.py tests/test_gpu_streams.py -x -q > gpurun_out/t_new_$TAG.log 2>&1; echo "new rc=$?"; tail -30 gpurun_out/t_new_$TAG.log
for i in 1 2; do timeout 300 python scripts/variants.py run 8192 base >> gpurun_out/var8192_$TAG.log 2>&1; done; cat gpurun_out/var8192_$TAG.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/t_all_$TAG.log 2>&1; echo "all rc=$?"; tail -5 gpurun_out/t_all_$TAG.log
