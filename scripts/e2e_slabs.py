"""e2e (host operands) at 16384^3 for several slab shapes (dev probe):
casc_gemm_fp64x2_host, 3 calls back to back per setting, CUDA events."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import casc_inputs as I
import paper_2303_04353_b200 as casc

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
d = I.make_config(4, m=n, n=n, k=n, seed=4)
h = [torch.from_numpy(np.ascontiguousarray(d[x])).pin_memory() for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
del d
oC = [torch.empty((n, n), dtype=torch.float64).pin_memory() for _ in range(2)]
oF = torch.empty((n, n), dtype=torch.uint8).pin_memory()
st = torch.cuda.current_stream()
for sr, sc in [(0, 0), (4096, 4096), (2048, 2368), (4096, 2368), (2048, 4736), (1024, 4736)]:
    call = lambda: casc.casc_gemm_fp64x2_host(*h, C_hi=oC[0], C_lo=oC[1], flags=oF, slab_rows=sr,
                                              slab_cols=sc, stream=st, sync=False)
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        call()
    e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    print(f"slabs {sr}x{sc}: {t:.1f} ms  {2*n**3/t/1e6:.1f} GFLOP/s", flush=True)
