"""Quick device timing of the C-ABI call at a few sizes (development probe)."""
import sys, json, torch
sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc

def t(n, reps=3):
    g = torch.Generator(device="cuda").manual_seed(0)
    A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A_lo = A_hi * 2.0**-54; B_lo = B_hi * 2.0**-54
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
    C_hi = torch.empty(n, n, dtype=torch.float64, device="cuda"); C_lo = torch.empty_like(C_hi)
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    for _ in range(2):
        casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C_hi, C_lo=C_lo, flags=fl, workspace=ws)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C_hi, C_lo=C_lo, flags=fl, workspace=ws); e1.record()
        e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    # packed-only (gemm kernel alone)
    pa = casc.casc_pack_a(A_hi, A_lo); pb = casc.casc_pack_b(B_hi, B_lo)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); casc.casc_gemm_packed(n, n, n, pa, pb, C_hi=C_hi, C_lo=C_lo, flags=fl); e1.record(); e1.synchronize()
    g_ms = e0.elapsed_time(e1)
    e0.record(); casc.casc_pack_a(A_hi, A_lo, packed=pa); casc.casc_pack_b(B_hi, B_lo, packed=pb); e1.record(); e1.synchronize()
    s_ms = e0.elapsed_time(e1)
    eff = 2 * n**3 / (best * 1e-3) / 1e9
    print(json.dumps({"n": n, "ms": best, "eff_gflops": eff, "frac_of_R/10": eff / 3706.7,
                      "gemm_kernel_ms": g_ms, "split_ms": s_ms,
                      "split_GBps": (16*2*n*n + 32*n*n + 56*n*n) / (s_ms*1e-3) / 1e9}), flush=True)

for n in [int(x) for x in sys.argv[1:]] or [1024, 4096, 8192]:
    t(n)
