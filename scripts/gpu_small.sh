#!/bin/bash
# small-problem breakdown: event timings, then the per-kernel launch list (ncu)
mkdir -p gpurun_out
python scripts/small_breakdown.py 512 1024 2048 > gpurun_out/small_breakdown.txt 2>&1; echo "breakdown rc=$?"
cat gpurun_out/small_breakdown.txt
python scripts/small_kernels.py 512 1024 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/small_launches.csv python scripts/small_kernels.py 512 1024 > gpurun_out/small_ncu.log 2>&1; echo "ncu rc=$?"
