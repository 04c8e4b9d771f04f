"""Time the simple path (casc_gemm_fp64x2_simple) against the fused path."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import casc_inputs as I
import paper_2303_04353_b200 as casc
n = int(sys.argv[1])
d = I.make_config(1, m=n, n=n, k=n)
A_hi, A_lo, B_hi, B_lo = (torch.from_numpy(d[x]).cuda() for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
out = {}
for name, fn in (("simple", casc.casc_gemm_fp64x2_simple), ("fused", casc.casc_gemm_fp64x2)):
    fn(A_hi, A_lo, B_hi, B_lo)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); C = fn(A_hi, A_lo, B_hi, B_lo); e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1)
    out[name] = {"ms": ms, "eff_gflops": 2 * n**3 / ms / 1e6, "launches": casc.casc_last_launch_count()}
# epilogue algorithmic bytes per panel launch: 32 B bins + 16 B C read (q>0) + 16 B C write + 2 B flags
out["epilogue_bytes_per_launch"] = 66 * n * n
out["slice_gemm_flops_per_launch"] = 2 * n * n * 256
print(json.dumps(out))
