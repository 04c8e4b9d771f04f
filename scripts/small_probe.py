import sys, json, torch
sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc
n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
g = torch.Generator(device="cuda").manual_seed(0)
A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
A_lo, B_lo = A_hi * 2.0**-54, B_hi * 2.0**-54
ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
i8ws = torch.empty(casc.casc_i8_workspace_bytes(n, n, n, 14), dtype=torch.uint8, device="cuda")
C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
def t(f, reps=20):
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
pa = casc.casc_pack_a(A_hi, A_lo); pb = casc.casc_pack_b(B_hi, B_lo)
i8pa = casc.casc_i8_pack(A_hi, A_lo, False, 14); i8pb = casc.casc_i8_pack(B_hi, B_lo, True, 14)
res = {
 "fp64_call": t(lambda: casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1], flags=fl, workspace=ws)),
 "fp64_pack_a": t(lambda: casc.casc_pack_a(A_hi, A_lo, packed=pa)),
 "fp64_gemm_packed": t(lambda: casc.casc_gemm_packed(n, n, n, pa, pb, C_hi=C[0], C_lo=C[1], flags=fl)),
 "i8_call": t(lambda: casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1], flags=fl, workspace=i8ws)),
 "i8_pack_a": t(lambda: casc.casc_i8_pack(A_hi, A_lo, False, 14, packed=i8pa)),
 "i8_gemm_packed": t(lambda: casc.casc_i8_gemm_packed(n, n, n, i8pa, i8pb, 14, C_hi=C[0], C_lo=C[1], flags=fl)),
}
print(json.dumps({k: round(v, 4) for k, v in res.items()}))
