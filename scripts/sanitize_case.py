"""Small end-to-end run of every entry point, for compute-sanitizer (one tool per call).
832x832x300: 169 tiles > 148 SMs, so the wave barrier, TMEM C and multi-panel paths run."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import casc_inputs as I
import paper_2303_04353_b200 as casc
d = I.make_config(1, m=832, n=832, k=300)
A_hi, A_lo, B_hi, B_lo = (torch.from_numpy(d[x]).cuda() for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
C = casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)
S = casc.casc_gemm_fp64x2_simple(A_hi[:70], A_lo[:70], B_hi[:, :90], B_lo[:, :90])
casc.casc_split_a(A_hi[:65], A_lo[:65]); casc.casc_split_b(B_hi[:, :70], B_lo[:, :70])
casc.casc_debug_bins(A_hi[:65], A_lo[:65], B_hi[:, :70], B_lo[:, :70], 1)
casc.casc_slice_product(A_hi[:33], A_lo[:33], B_hi[:, :40], B_lo[:, :40], 2, 5, 1)
torch.cuda.synchronize()
print("sanitize case ok", float(C[0].abs().sum()), float(S[0].abs().sum()))
