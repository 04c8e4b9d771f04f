"""NEXT-1 on the GPU: the paper's accuracy claims (§5.2) for 240^3 products.

* uniform [-1, 1] data: the cascaded GEMM is at least as accurate as plain
  FP64x2 (ORACLE-DD) in the max componentwise relative error (P:L3548-3553
  "our approach tends to be more accurate");
* ill-conditioned data (t = 1e-9, 1e-14, 1e-19): "the accuracy of the cascaded
  multiply in these experiments is vastly superior to that of FP64x2"
   — max relative error of the cascade below ORACLE-DD's;
* wide-range data behaves like well-conditioned data: within
  the north-star bound everywhere.
Errors are against the exact product (superaccumulator)."""

import numpy as np
import pytest

from casc_inputs import paper_generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def casc():
    import torch
    assert torch.cuda.is_available()
    import paper_2303_04353_b200 as casc
    return casc


def _errors(orc, casc, d):
    import torch
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    g = [x.cpu().numpy() for x in casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]),
                                                          T(d["B_hi"]), T(d["B_lo"]))]
    o = orc.dd_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    n = d["m"]
    ii, jj = np.meshgrid(np.arange(n), np.arange(d["n"]), indexing="ij")
    out = []
    for C_hi, C_lo in ((g[0], g[1]), o):
        r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                              C_hi, C_lo)
        ex = np.abs(r["ex_hi"])
        out.append((np.abs(r["err"]) / ex, r))
    return out[0], out[1], g[2]


def test_uniform_240(orc, casc):
    Ah, Al = G.gen_uniform_dd(100, 240, 240, stream=30)
    Bh, Bl = G.gen_uniform_dd(200, 240, 240, stream=32)
    (rc, r), (rd, _), fl = _errors(orc, casc, dict(A_hi=Ah, A_lo=Al, B_hi=Bh, B_lo=Bl, m=240,
                                                     n=240, k=240))
    assert rc.max() <= rd.max()
    assert np.all(np.abs(r["err"]) <= orc.north_star_bound(240, r["absab"]))
    assert fl.sum() == 0


@pytest.mark.parametrize("t", [1e-9, 1e-14, 1e-19])
def test_illcond_240(orc, casc, t):
    d = G.gen_illcond(400, 240, t)
    (rc, _), (rd, _), _ = _errors(orc, casc, d)
    assert rc.max() < rd.max()


def test_widerange_240(orc, casc):
    d = G.gen_widerange(300, 240, 240, 240)
    (rc, r), (rd, _), fl = _errors(orc, casc, d)
    assert np.all(np.abs(r["err"]) <= orc.north_star_bound(240, r["absab"]))
