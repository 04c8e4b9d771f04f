"""Write-safety without compute-sanitizer (closed on this GPU pool): every
output lives inside a larger buffer whose margins (before, after, and the gap
columns of a strided leading dimension) hold a sentinel; after each entry
point runs on ragged shapes, all sentinels must be intact and every output
element must have been written (finite, not the sentinel)."""

import numpy as np
import pytest

import casc_inputs as I

pytestmark = pytest.mark.gpu

SENT = -7.25e300


def _boxed(torch, m, n, gap=3, pad=4096):
    """An m x n view with ld = n + gap inside a sentinel-filled buffer."""
    ld = n + gap
    buf = torch.full((pad + m * ld + pad,), SENT, dtype=torch.float64, device="cuda")
    view = buf[pad:pad + m * ld].view(m, ld)[:, :n]
    return buf, view


def _check(buf, view, m, n, gap=3, pad=4096, tri=None):
    b = buf.cpu().numpy()
    assert np.all(b[:pad] == SENT) and np.all(b[-pad:] == SENT), "write outside the matrix"
    inner = b[pad:pad + m * (n + gap)].reshape(m, n + gap)
    assert np.all(inner[:, n:] == SENT), "write into the leading-dimension gap"
    v = inner[:, :n]
    mask = np.ones((m, n), bool) if tri is None else tri
    assert np.all(np.isfinite(v[mask])) and np.all(v[mask] != SENT), "element not written"
    assert np.all(v[~mask] == SENT), "write outside the triangle"


@pytest.mark.parametrize("m,n,k", [(130, 257, 300), (65, 1000, 8192 + 40), (300, 64, 129)])
def test_output_canaries(m, n, k):
    import torch

    import paper_2303_04353_b200 as casc
    d = I.make_config(1, m=m, n=n, k=k, seed=101)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    for fn in (casc.casc_gemm_fp64x2, casc.casc_i8_gemm_fp64x2):
        bh, vh = _boxed(torch, m, n)
        bl, vl = _boxed(torch, m, n)
        fl = torch.full((m, n), 9, dtype=torch.uint8, device="cuda")
        fn(A_hi, A_lo, B_hi, B_lo, C_hi=vh, C_lo=vl, flags=fl)
        torch.cuda.synchronize()
        _check(bh, vh, m, n)
        _check(bl, vl, m, n)
        assert np.all(fl.cpu().numpy() <= 1)
    # BLAS-style update (beta != 0 reads C) and SYRK (one triangle) on both cascades
    for ex in (casc.casc_gemm_fp64x2_ex, casc.casc_i8_gemm_fp64x2_ex):
        bh, vh = _boxed(torch, m, n)
        bl, vl = _boxed(torch, m, n)
        vh.fill_(0.5)
        vl.fill_(0.0)
        ex("N", "N", 2.0, A_hi, A_lo, B_hi, B_lo, 1.0, vh, vl)
        torch.cuda.synchronize()
        _check(bh, vh, m, n)
        _check(bl, vl, m, n)
    s = min(m, 300)
    for syrk in (casc.casc_syrk_fp64x2, casc.casc_i8_syrk_fp64x2):
        for uplo in ("L", "U"):
            bh, vh = _boxed(torch, s, s)
            bl, vl = _boxed(torch, s, s)
            syrk(uplo, "N", 1.0, A_hi[:s], A_lo[:s], 0.0, vh, vl)
            torch.cuda.synchronize()
            tri = np.tril(np.ones((s, s), bool)) if uplo == "L" else np.triu(np.ones((s, s), bool))
            _check(bh, vh, s, s, tri=tri)
            _check(bl, vl, s, s, tri=tri)


def test_trsm_and_host_canaries():
    """TRSM writes only its B (ragged m, strided ldb); the host-operand entry
    writes only its host C block (sentinels in pinned host memory)."""
    import torch

    import paper_2303_04353_b200 as casc
    m, n = 300, 37
    rng = np.random.default_rng(5)
    L = np.tril(rng.uniform(-1, 1, (m, m)) / m) + np.diag(1.0 + rng.uniform(0, 1, m))
    bh, vh = _boxed(torch, m, n)
    bl, vl = _boxed(torch, m, n)
    vh.copy_(torch.from_numpy(rng.uniform(-1, 1, (m, n))).cuda())
    vl.zero_()
    Lh = torch.from_numpy(L).cuda()
    casc.casc_trsm_fp64x2("L", "N", 1.0, Lh, Lh * 2.0 ** -54, vh, vl)
    torch.cuda.synchronize()
    _check(bh, vh, m, n)
    _check(bl, vl, m, n)
    # host-operand entry: C as a window of a sentinel-filled pinned host buffer
    d = I.make_config(2, m=200, n=150, k=300, seed=7)
    P = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hb = torch.full((400, 160), SENT, dtype=torch.float64).pin_memory()
    lb = torch.full((400, 160), SENT, dtype=torch.float64).pin_memory()
    casc.casc_gemm_fp64x2_host(P(d["A_hi"]), P(d["A_lo"]), P(d["B_hi"]), P(d["B_lo"]),
                               C_hi=hb[100:300, 5:155], C_lo=lb[100:300, 5:155], want_flags=False,
                               slab_rows=64, slab_cols=64)
    for b in (hb.numpy(), lb.numpy()):
        inside = np.zeros((400, 160), bool)
        inside[100:300, 5:155] = True
        assert np.all(b[~inside] == SENT) and np.all(np.isfinite(b[inside]))
