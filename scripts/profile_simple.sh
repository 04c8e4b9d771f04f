#!/bin/bash
# Simple path (§4.2) timing + ncu of its standalone epilogue and one slice GEMM (4096^3).
mkdir -p gpurun_out
TAG=${1:-r01}
CMD="python scripts/time_simple.py 4096"
$CMD > gpurun_out/simple_time_$TAG.json 2>&1 && cat gpurun_out/simple_time_$TAG.json && \
ncu --set full --clock-control none -k regex:casc_epilogue -s 3 -c 1 -o gpurun_out/prof_epilogue_$TAG $CMD > gpurun_out/ncu_epi_$TAG.log 2>&1; echo "ncu epi rc=$?"
$CMD > /dev/null 2>&1 && \
ncu --set full --clock-control none -k regex:slice_gemm -s 20 -c 1 -o gpurun_out/prof_slice_$TAG $CMD > gpurun_out/ncu_slice_$TAG.log 2>&1; echo "ncu slice rc=$?"
