#!/bin/bash
# ncu evidence for one round tag: launch list of the headline step (FP64 cascade
# only, cfg4) and one --set full capture of each hot kernel of the bench.
# Usage: bash scripts/gpu_ncu.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-int8 --no-next4 --no-small"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
CMD4="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4 --no-small"
$CMD4 > gpurun_out/plain4_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:casc_gemm_kernel -s 6 -c 1 -o gpurun_out/prof_gemm_$TAG $CMD4 > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:split -s 6 -c 2 -o gpurun_out/prof_split_$TAG $CMD4 > gpurun_out/ncu_split_$TAG.log 2>&1; echo "ncu split rc=$?"
ncu --set full --clock-control none --import-source on -k regex:i8_gemm -s 3 -c 1 -o gpurun_out/prof_i8gemm_$TAG $CMD4 > gpurun_out/ncu_i8gemm_$TAG.log 2>&1; echo "ncu i8 gemm rc=$?"
