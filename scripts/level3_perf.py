"""Level-3 routines at n^3 on one B200 (dev probe): TRMM (banded), SYMM, SYR2K,
right-side TRSM, vs the GEMM; CUDA events, device-resident operands."""
import sys
import torch
sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
Al, Bl = A * 2.0**-54, B * 2.0**-54
L = torch.tril(A / n) + torch.diag(2.0 + A.diagonal().abs())
Ll = L * 2.0**-54
C, Cl = torch.zeros_like(A), torch.zeros_like(A)
X, Xl = torch.empty_like(A), torch.empty_like(A)


def t(f, reps=2):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def cp():
    X.copy_(B)
    Xl.copy_(Bl)


res = {
    "gemm": t(lambda: casc.casc_gemm_fp64x2_ex("N", "N", 1.0, A, Al, B, Bl, 0.0, C, Cl)),
    "trmm_L": t(lambda: (cp(), casc.casc_trmm_fp64x2("L", "L", "N", 1.0, L, Ll, X, Xl))),
    "trmm_R_T": t(lambda: (cp(), casc.casc_trmm_fp64x2("R", "L", "N", 1.0, L, Ll, X, Xl, trans="T"))),
    "symm": t(lambda: casc.casc_symm_fp64x2("L", "L", 1.0, A, Al, B, Bl, 0.0, C, Cl)),
    "syr2k": t(lambda: casc.casc_syr2k_fp64x2("L", "N", 1.0, A, Al, B, Bl, 0.0, C, Cl)),
    "syrk": t(lambda: casc.casc_syrk_fp64x2("L", "N", 1.0, A, Al, 0.0, C, Cl)),
    "trsm_L": t(lambda: (cp(), casc.casc_trsm_fp64x2("L", "N", 1.0, L, Ll, X, Xl))),
    "trsm_R": t(lambda: (cp(), casc.casc_trsm_fp64x2_right("L", "N", 1.0, L, Ll, X, Xl, trans="T"))),
}
print({k: round(v, 2) for k, v in res.items()})
