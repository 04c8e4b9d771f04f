"""Do the C-ABI entry points capture into a CUDA graph (torch.cuda.graph) and
replay bitwise?  Times eager vs graph replay for small problems."""
import json
import sys

import torch

sys.path.insert(0, ".")
import paper_2303_04353_b200 as casc  # noqa: E402

out = {}
for n in (64, 256, 1024):
    g = torch.Generator(device="cuda").manual_seed(0)
    A_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    B_hi = torch.rand(n, n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    A_lo, B_lo = A_hi * 2.0**-54, B_hi * 2.0**-54
    C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fl = torch.empty(n, n, dtype=torch.uint8, device="cuda")
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")
    i8ws = torch.empty(casc.casc_i8_workspace_bytes(n, n, n, 14), dtype=torch.uint8, device="cuda")
    C8 = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(2)]
    fl8 = torch.empty(n, n, dtype=torch.uint8, device="cuda")

    def step():
        casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1], flags=fl, workspace=ws)
        casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C8[0], C_lo=C8[1], flags=fl8,
                                 workspace=i8ws)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    ref = [t.clone() for t in (C[0], C[1], fl, C8[0], C8[1], fl8)]
    graph = torch.cuda.CUDAGraph()
    try:
        with torch.cuda.graph(graph):
            step()
    except Exception as ex:  # noqa: BLE001
        out[n] = {"capture": "failed: " + str(ex)[:200]}
        continue
    for t in (C[0], C[1], C8[0], C8[1]):
        t.fill_(float("nan"))
    graph.replay()
    torch.cuda.synchronize()
    same = all(torch.equal(a.view(torch.uint8) if a.dtype == torch.float64 else a,
                           b.view(torch.uint8) if b.dtype == torch.float64 else b)
               for a, b in zip((C[0], C[1], fl, C8[0], C8[1], fl8), ref))

    def timeit(f, reps=20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(reps):
            f()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out[n] = {"replay_bitwise": same, "eager_ms": timeit(step), "graph_ms": timeit(graph.replay)}
print(json.dumps(out))
