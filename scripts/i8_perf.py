"""Device timing of the INT8 cascade's C-ABI call (development probe).
Usage: python scripts/i8_perf.py [n ...] [--y Y] [--reps R]"""
import argparse
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("sizes", nargs="*", type=int, default=[1024, 4096, 8192])
ap.add_argument("--y", type=int, default=14)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()

for n in a.sizes:
    g = torch.Generator(device="cuda").manual_seed(0)
    A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A_lo = A_hi * 2.0**-54
    B_lo = B_hi * 2.0**-54
    ws = torch.empty(casc.casc_i8_workspace_bytes(n, n, n, a.y), dtype=torch.uint8, device="cuda")
    C_hi = torch.empty(n, n, dtype=torch.float64, device="cuda")
    C_lo = torch.empty_like(C_hi)
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    call = lambda: casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, y=a.y, C_hi=C_hi, C_lo=C_lo,
                                            flags=fl, workspace=ws)
    for _ in range(2):
        call()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(a.reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    eff = 2 * n**3 / (best * 1e-3) / 1e9
    prods = a.y * (a.y + 1) // 2
    print(json.dumps({"n": n, "y": a.y, "ms": best, "eff_gflops": eff,
                      "int8_tops": prods * 2 * n**3 / (best * 1e-3) / 1e12}), flush=True)
