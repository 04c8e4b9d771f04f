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
