"""e2e (host operands) at 16384^3, both cascades, default blocks (first slabs
of 1024 rows / columns) vs uniform blocks (dev probe), 3 calls back to back."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import casc_inputs as I
import paper_2303_04353_b200 as casc

n = 16384
d = I.make_config(4, m=n, n=n, k=n, seed=4)
h = [torch.from_numpy(np.ascontiguousarray(d[x])).pin_memory() for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
del d
oC = [torch.empty((n, n), dtype=torch.float64).pin_memory() for _ in range(2)]
oF = torch.empty((n, n), dtype=torch.uint8).pin_memory()
st = torch.cuda.current_stream()
for name, fn, slabs in [("fp64 default", casc.casc_gemm_fp64x2_host, (0, 0)),
                        ("fp64 uniform 4096x2368", casc.casc_gemm_fp64x2_host, (4096, 2368)),
                        ("i8 default", casc.casc_i8_gemm_fp64x2_host, (0, 0)),
                        ("i8 uniform 4096x4096", casc.casc_i8_gemm_fp64x2_host, (4096, 4096))]:
    call = lambda: fn(*h, C_hi=oC[0], C_lo=oC[1], flags=oF, slab_rows=slabs[0],
                      slab_cols=slabs[1], stream=st, sync=False)
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(3):
        call()
    e1.record(st)
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 3
    print(f"{name}: {t:.1f} ms  {2*n**3/t/1e6:.1f} GFLOP/s", flush=True)
