#!/bin/bash
# One GPU session: tests, bench lines, ncu launch list + full captures.
# Usage: bash scripts/gpu_round.sh <tag> [skip_tests]
TAG=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
if [ -z "$2" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_$TAG.log
fi
python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/bench_cfg1_$TAG.json 2> gpurun_out/bench_cfg1_$TAG.err; echo "bench cfg1 rc=$?"
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
cat gpurun_out/bench_$TAG.json
python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
# launch list of the bench command (plain run first, then under ncu)
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
# full captures on the bench workload (cfg4): the fused GEMM and the split kernels
CMD4="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD4 > gpurun_out/plain4_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:casc_gemm -s 3 -c 1 -o gpurun_out/prof_gemm_$TAG $CMD4 > gpurun_out/ncu_gemm_$TAG.log 2>&1; echo "ncu gemm rc=$?"
$CMD4 > gpurun_out/plain5_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:split -s 3 -c 1 -o gpurun_out/prof_split_$TAG $CMD4 > gpurun_out/ncu_split_$TAG.log 2>&1; echo "ncu split rc=$?"
$CMD4 > gpurun_out/plain6_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:i8_gemm -s 3 -c 1 -o gpurun_out/prof_i8gemm_$TAG $CMD4 > gpurun_out/ncu_i8gemm_$TAG.log 2>&1; echo "ncu i8 gemm rc=$?"
$CMD4 > gpurun_out/plain7_$TAG.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:i8_digits -s 6 -c 2 -o gpurun_out/prof_i8split_$TAG $CMD4 > gpurun_out/ncu_i8split_$TAG.log 2>&1; echo "ncu i8 split rc=$?"
