# cuBLAS DGEMM throughput (context only, never on the hot path): t_DGEMM for the
# paper's slowdown ratio t/t_DGEMM.
import json, torch
res = {}
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(5 if n < 16384 else 3):
        e0.record(); torch.matmul(a, b); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = {"ms": best, "tflops": 2 * n**3 / (best * 1e-3) / 1e12}
    del a, b
print(json.dumps({"cublas_dgemm": res}))
