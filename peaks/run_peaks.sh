#!/bin/bash
# Runs the FP64 peak microbenchmark and the cuBLAS DGEMM context timing with
# nvidia-smi clock sampling; results land in gpurun_out/peaks_*.
set -e
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/peaks_clocks.csv &
SMI=$!
./peaks/mma_layout_probe | tee gpurun_out/peaks_layout.json
./peaks/fp64_peak | tee gpurun_out/peaks_fp64.json
python peaks/dgemm_ctx.py | tee gpurun_out/peaks_dgemm.json
kill $SMI || true
