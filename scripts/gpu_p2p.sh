#!/bin/bash
# the peer-memory exchange on the one GPU: two processes (CUDA IPC within the
# device), then the bench's N > 1 path in plumbing mode (NOT a measurement)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multiproc.py -x -q -p no:cacheprovider > gpurun_out/t_p2p.log 2>&1; echo "multiproc rc=$?"; tail -3 gpurun_out/t_p2p.log
CASC_BENCH_PLUMBING=1 timeout 900 python bench.py --gpus 2 --config 1 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/plumb2.json 2> gpurun_out/plumb2.err; echo "plumbing rc=$?"; tail -c 1500 gpurun_out/plumb2.json; grep -v NCCL gpurun_out/plumb2.err | tail -5
