"""Device timing of casc_syrk_fp64x2 against casc_gemm_fp64x2_ex on the same
product (development probe): python scripts/syrk_perf.py [n] [k]"""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
k = int(sys.argv[2]) if len(sys.argv) > 2 else n
g = torch.Generator(device="cuda").manual_seed(0)
A_hi = torch.rand(n, k, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
A_lo = A_hi * 2.0**-54
C_hi = torch.zeros(n, n, dtype=torch.float64, device="cuda")
C_lo = torch.zeros_like(C_hi)
ws = torch.empty(casc.casc_workspace_bytes(n, n, k), dtype=torch.uint8, device="cuda")
out = {"n": n, "k": k}
for name, call in [
        ("syrk", lambda: casc.casc_syrk_fp64x2("L", "N", 1.0, A_hi, A_lo, 0.0, C_hi, C_lo,
                                               workspace=ws)),
        ("gemm_ex", lambda: casc.casc_gemm_fp64x2_ex("N", "T", 1.0, A_hi, A_lo, A_hi, A_lo, 0.0,
                                                     C_hi, C_lo, workspace=ws)),
        ("i8_syrk", lambda: casc.casc_i8_syrk_fp64x2("L", "N", 1.0, A_hi, A_lo, 0.0, C_hi, C_lo)),
        ("i8_gemm_ex", lambda: casc.casc_i8_gemm_fp64x2_ex("N", "T", 1.0, A_hi, A_lo, A_hi, A_lo,
                                                           0.0, C_hi, C_lo))]:
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        call()
    e1.record()
    torch.cuda.synchronize()
    out[name + "_ms"] = e0.elapsed_time(e1) / 2
# SYRK convention: n(n+1)k useful FP64x2 multiply-adds ~ n^2 k
out["syrk_eff_gflops_n2k"] = (n * (n + 1) * k) / (out["syrk_ms"] * 1e-3) / 1e9
out["gemm_eff_gflops_2n2k"] = 2.0 * n * n * k / (out["gemm_ex_ms"] * 1e-3) / 1e9
print(json.dumps(out))
