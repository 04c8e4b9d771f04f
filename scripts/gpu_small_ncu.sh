#!/bin/bash
# one full ncu capture of the split-mode fused GEMM at 1024^3 (and tile mode at 2048^3)
mkdir -p gpurun_out
python scripts/small_kernels.py 1024 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:casc_gemm_kernel -s 2 -c 1 -o gpurun_out/prof_split1024 python scripts/small_kernels.py 1024 > gpurun_out/ncu_s1024.log 2>&1; echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:casc_gemm_kernel -s 2 -c 1 -o gpurun_out/prof_tile2048 python scripts/small_kernels.py 2048 > gpurun_out/ncu_t2048.log 2>&1; echo "ncu2 rc=$?"
