"""Per-rank compute of the sharded cfg4 step on ONE GPU (dev probe; not a
scaling measurement: no exchange runs, nothing crosses NVLink).

For N in 1, 2, 4, 8 and a few ranks r, the kernels rank r launches in
ShardedCascGemm's overlapped step are timed back to back on one B200 (CUDA
events): pack A rows [r0, r1), pack the own column slab of B, GEMM over the own
columns, GEMM over the other columns (their packed slices prepared outside the
timed region, standing in for the all-gather's result).  The ratio
t(1) / (N * max_r t_rank(N)) is the efficiency the COMPUTE of the sharded step
allows (tile-wave quantisation of the two launches, per-rank split work);
the exchange's own cost and its overlap are not in it.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import casc_inputs as I
import paper_2303_04353_b200 as casc
from paper_2303_04353_b200.multigpu import col_slab, row_shard

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
m = k = n
d = I.make_config(4, m=m, n=n, k=k, seed=4)
A_hi, A_lo, B_hi, B_lo = (torch.from_numpy(np.ascontiguousarray(d[x])).cuda()
                          for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
del d
blk = casc.casc_packed_b_block_bytes(k)


def rank_time(N, r, reps=2):
    r0, r1 = row_shard(m, N, r)
    c0, c1, per = col_slab(n, N, r)
    mloc = r1 - r0
    full = torch.empty(per * N * blk, dtype=torch.uint8, device="cuda")
    for q in range(N):  # the other ranks' slabs: what the all-gather would deliver
        a0, a1 = col_slab(n, N, q)[:2]
        if q != r and a1 > a0:
            casc.casc_pack_b(B_hi[:, a0:a1].contiguous(), B_lo[:, a0:a1].contiguous(),
                             packed=full[q * per * blk:q * per * blk + -(-(a1 - a0) // 64) * blk])
    Ar_hi, Ar_lo = A_hi[r0:r1].contiguous(), A_lo[r0:r1].contiguous()
    Bs_hi, Bs_lo = B_hi[:, c0:c1].contiguous(), B_lo[:, c0:c1].contiguous()
    C_hi = torch.empty((mloc, n), dtype=torch.float64, device="cuda")
    C_lo = torch.empty((mloc, n), dtype=torch.float64, device="cuda")
    fl = torch.empty((mloc, n), dtype=torch.uint8, device="cuda")
    pa = casc.casc_pack_a(Ar_hi, Ar_lo)

    def gemm(col0, col1):
        if col1 > col0:
            casc.casc_gemm_packed(mloc, col1 - col0, k, pa, full[(col0 // 64) * blk:],
                                  C_hi=C_hi[:, col0:col1], C_lo=C_lo[:, col0:col1],
                                  flags=fl[:, col0:col1])

    def step():
        casc.casc_pack_a(Ar_hi, Ar_lo, packed=pa)
        own = full[r * per * blk:r * per * blk + -(-(c1 - c0) // 64) * blk]
        casc.casc_pack_b(Bs_hi, Bs_lo, packed=own)
        if N == 1:
            gemm(0, n)
            return
        gemm(c0, c1)
        gemm(c1, n)
        gemm(0, c0)

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def rank_time_with_copies(N, r, reps=2):
    """Rank r's step at N with the p2p exchange's copy-engine traffic running
    beside the own-slab GEMM: the same bytes (the other N-1 packed slabs) copied
    device to device on two copy streams (cudaMemcpyAsync, no SM), each slab's
    GEMM waiting for its copy -- the compute-side cost of the overlap on one GPU
    (the NVLink link itself is not in it)."""
    r0, r1 = row_shard(m, N, r)
    c0, c1, per = col_slab(n, N, r)
    mloc = r1 - r0
    full = torch.empty(per * N * blk, dtype=torch.uint8, device="cuda")
    src = torch.empty_like(full)  # stands in for the peers' exported buffers
    for q in range(N):
        a0, a1 = col_slab(n, N, q)[:2]
        casc.casc_pack_b(B_hi[:, a0:a1].contiguous(), B_lo[:, a0:a1].contiguous(),
                         packed=src[q * per * blk:q * per * blk + -(-(a1 - a0) // 64) * blk])
    Ar_hi, Ar_lo = A_hi[r0:r1].contiguous(), A_lo[r0:r1].contiguous()
    Bs_hi, Bs_lo = B_hi[:, c0:c1].contiguous(), B_lo[:, c0:c1].contiguous()
    C_hi = torch.empty((mloc, n), dtype=torch.float64, device="cuda")
    C_lo = torch.empty((mloc, n), dtype=torch.float64, device="cuda")
    fl = torch.empty((mloc, n), dtype=torch.uint8, device="cuda")
    pa = casc.casc_pack_a(Ar_hi, Ar_lo)
    cs = [torch.cuda.Stream() for _ in range(2)]
    evq = [torch.cuda.Event() for _ in range(N)]
    cur = torch.cuda.current_stream()

    def gemm(col0, col1):
        if col1 > col0:
            casc.casc_gemm_packed(mloc, col1 - col0, k, pa, full[(col0 // 64) * blk:],
                                  C_hi=C_hi[:, col0:col1], C_lo=C_lo[:, col0:col1],
                                  flags=fl[:, col0:col1])

    def step():
        casc.casc_pack_a(Ar_hi, Ar_lo, packed=pa)
        casc.casc_pack_b(Bs_hi, Bs_lo,
                         packed=full[r * per * blk:r * per * blk + -(-(c1 - c0) // 64) * blk])
        started = torch.cuda.Event()
        started.record(cur)
        order = [(r + i) % N for i in range(1, N)]
        for i, q in enumerate(order):
            s = cs[i % 2]
            s.wait_event(started)
            a0, a1 = col_slab(n, N, q)[:2]
            nb = -(-(a1 - a0) // 64) * blk
            casc.casc_copy_async(full.data_ptr() + q * per * blk, src.data_ptr() + q * per * blk,
                                 nb, stream=s)
            evq[q].record(s)
        gemm(c0, c1)
        for q in order:
            cur.wait_event(evq[q])
            gemm(*col_slab(n, N, q)[:2])

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"n": n, "note": __doc__.split("\n\n")[0]}
t1 = rank_time(1, 0)
out["t1_ms"] = t1
for N in (2, 4, 8):
    ranks = sorted({0, N // 2, N - 1})
    ts = {r: rank_time(N, r) for r in ranks}
    tc = rank_time_with_copies(N, N - 1)
    out[f"N{N}"] = {"rank_ms": ts, "compute_efficiency": t1 / (N * max(ts.values())),
                    "rank_ms_with_ce_copies": {N - 1: tc},
                    "ce_copy_bytes_per_rank": (N - 1) * col_slab(n, N, 0)[2] * blk}
    print(N, out[f"N{N}"], flush=True)
print(json.dumps(out))
