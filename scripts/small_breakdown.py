"""Where the time of a small FP64-cascade call goes (dev probe): for each n,
20 calls back to back of (a) the whole casc_gemm_fp64x2_ws call, (b) the two
pack (split) calls alone, (c) casc_gemm_packed alone (split mode and, with
CASC_SPLIT_MODE=0, the tile mode), median of 5 runs, CUDA events."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import casc_inputs as I
import paper_2303_04353_b200 as casc


def timed(fn, reps=20, runs=5):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(runs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1) / reps)
    return float(np.median(out))


for n in [int(x) for x in sys.argv[1:]] or [512, 1024, 2048]:
    d = I.make_config(1, m=n, n=n, k=n, seed=1)
    A_hi, A_lo, B_hi, B_lo = (torch.from_numpy(np.ascontiguousarray(d[x])).cuda()
                              for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
    C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    pa = casc.casc_pack_a(A_hi, A_lo)
    pb = casc.casc_pack_b(B_hi, B_lo)
    ideal = 2 * n ** 3 / (37.109e12 / 10) * 1e3
    r = {"n": n, "ideal_ms_R/10": ideal}
    r["full"] = timed(lambda: casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1],
                                                    flags=fl, workspace=ws))
    r["packs"] = timed(lambda: (casc.casc_pack_a(A_hi, A_lo, packed=pa),
                                casc.casc_pack_b(B_hi, B_lo, packed=pb)))
    r["gemm_packed"] = timed(lambda: casc.casc_gemm_packed(n, n, n, pa, pb, C_hi=C[0], C_lo=C[1],
                                                           flags=fl))
    os.environ["CASC_SPLIT_MODE"] = "0"
    r["gemm_packed_tilemode"] = timed(lambda: casc.casc_gemm_packed(n, n, n, pa, pb, C_hi=C[0],
                                                                    C_lo=C[1], flags=fl))
    r["full_tilemode"] = timed(lambda: casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0],
                                                             C_lo=C[1], flags=fl, workspace=ws))
    del os.environ["CASC_SPLIT_MODE"]
    r["frac_full"] = ideal / r["full"]
    print({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}, flush=True)
