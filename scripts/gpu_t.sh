#!/bin/bash
# run given pytest targets on the GPU box; log to gpurun_out/t_<tag>.log
TAG=$1; shift
mkdir -p gpurun_out
timeout 1800 python -m pytest "$@" -x -q > gpurun_out/t_$TAG.log 2>&1; echo "rc=$?"; grep -E "^E |passed|failed" gpurun_out/t_$TAG.log | head -20
