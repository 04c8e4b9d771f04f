"""Per-kernel view of a small FP64-cascade call (dev probe, run under ncu
--metrics gpu__time_duration.sum): a few casc_gemm_fp64x2_ws calls at n^3."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import casc_inputs as I
import paper_2303_04353_b200 as casc
for n in [int(x) for x in sys.argv[1:]] or [1024, 512]:
    d = I.make_config(1, m=n, n=n, k=n, seed=1)
    A_hi, A_lo, B_hi, B_lo = (torch.from_numpy(np.ascontiguousarray(d[x])).cuda()
                              for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
    C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1], flags=fl, workspace=ws)
    torch.cuda.synchronize()
