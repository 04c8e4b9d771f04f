#!/bin/bash
mkdir -p gpurun_out
for n in 8192 16384; do for ws in 0 1; do echo "n=$n ws=$ws $(CASC_WAVE_SYNC=$ws python scripts/variants.py one $n)"; done; done
for ws in 0 1; do
  CASC_WAVE_SYNC=$ws python scripts/variants.py one 8192 > /dev/null && \
  CASC_WAVE_SYNC=$ws ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:casc_gemm -c 2 python scripts/variants.py one 8192 2>&1 | grep -E "dram__|gpu__time|lts__" | tail -5
done
