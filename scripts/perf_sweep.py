"""Size sweep in the paper's terms (its Fig. perf: cascaded FP64x2 GEMM time
divided by DGEMM time, 10-13x on one x86 core, ideal 10x):
square n, device-resident operands, CUDA events: best of 3 single calls after
warm-up, and (round 2) the mean of 10 calls back to back; nvidia-smi clocks
sampled during the sweep (bench.py's ClockSampler) and written with the rows.
cuBLAS DGEMM (torch.matmul, float64) is a timing reference only.

    python scripts/perf_sweep.py [--out profiles/.../perf_sweep.json]"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402
from bench import ClockSampler  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="256,512,1024,2048,4096,8192,16384")
ap.add_argument("--out", default=None)
a = ap.parse_args()


def steady(f, reps=10):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def best(f, reps=3):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


rows = []
cs = ClockSampler(None).__enter__()
for n in (int(x) for x in a.sizes.split(",")):
    g = torch.Generator(device="cuda").manual_seed(0)
    A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A_lo, B_lo = A_hi * 2.0**-54, B_hi * 2.0**-54
    C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
    ws8 = torch.empty(casc.casc_i8_workspace_bytes(n, n, n, 14), dtype=torch.uint8, device="cuda")
    t_c = best(lambda: casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1],
                                             flags=fl, workspace=ws))
    t_i8 = best(lambda: casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1],
                                                 flags=fl, workspace=ws8))
    t_d = best(lambda: torch.matmul(A_hi, B_hi, out=C[0]))
    reps = 10 if n <= 4096 else 2
    t_cs = steady(lambda: casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1],
                                                flags=fl, workspace=ws), reps)
    t_i8s = steady(lambda: casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1],
                                                    flags=fl, workspace=ws8), reps)
    f = 2.0 * n**3
    rows.append({"n": n, "cascade_ms": t_c, "int8_cascade_ms": t_i8, "dgemm_ms": t_d,
                 "cascade_gflops": f / t_c / 1e6, "int8_cascade_gflops": f / t_i8 / 1e6,
                 "dgemm_gflops": f / t_d / 1e6, "cascade_over_dgemm": t_c / t_d,
                 "int8_cascade_over_dgemm": t_i8 / t_d,
                 "cascade_frac_of_R_over_10": f / t_c / 1e6 / 3710.9,
                 "cascade_ms_back_to_back": t_cs, "int8_cascade_ms_back_to_back": t_i8s,
                 "cascade_frac_of_R_over_10_back_to_back": f / t_cs / 1e6 / 3710.9})
    print(json.dumps(rows[-1]), flush=True)
    del A_hi, B_hi, A_lo, B_lo, C, fl, ws, ws8
    torch.cuda.empty_cache()
cs.__exit__()
clocks = cs.summary()
print(json.dumps({"clocks": clocks}), flush=True)
if a.out:
    with open(a.out, "w") as fh:
        json.dump({"rows": rows, "clocks": clocks}, fh, indent=1)
