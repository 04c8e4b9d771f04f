"""Device timing of casc_trsm_fp64x2 (development probe): python scripts/trsm_perf.py [m] [n]
Effective FP64x2 GFLOP/s by the TRSM convention m^2 n / t."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402

args = [x for x in sys.argv[1:] if not x.startswith("--")]
m = int(args[0]) if args else 8192
n = int(args[1]) if len(args) > 1 else m
g = torch.Generator(device="cuda").manual_seed(0)
A_hi = torch.tril(torch.rand(m, m, dtype=torch.float64, device="cuda", generator=g) * 2 - 1) / m
A_hi += torch.diag(1.0 + torch.rand(m, dtype=torch.float64, device="cuda", generator=g))
A_lo = A_hi * 2.0**-54
B0 = torch.rand(m, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B_hi, B_lo = B0.clone(), B0 * 2.0**-54
fn = casc.casc_i8_trsm_fp64x2 if "--i8" in sys.argv else casc.casc_trsm_fp64x2
call = lambda: fn("L", "N", 1.0, A_hi, A_lo, B_hi, B_lo)
call()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
call()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
print(json.dumps({"m": m, "n": n, "ms": ms, "eff_gflops_m2n": m * m * n / (ms * 1e-3) / 1e9,
                  "frac_of_R_over_10": m * m * n / (ms * 1e-3) / 1e9 / 3710.9}))
