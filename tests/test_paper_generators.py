"""NEXT-1 generators (CPU): the paper's wide-range and ill-conditioned inputs
(§5.2), pinned against exact arithmetic."""

import random
from fractions import Fraction as F

import numpy as np

from casc_inputs import paper_generators as G


def test_dd_helpers_exact():
    rng = random.Random(3)
    for _ in range(3000):
        a = rng.uniform(-1, 1) * 2.0 ** rng.randint(-100, 100)
        b = rng.uniform(-1, 1) * 2.0 ** rng.randint(-100, 100)
        s, e = G._two_sum(np.float64(a), np.float64(b))
        assert F(float(s)) + F(float(e)) == F(a) + F(b)
        p, e = G._two_prod(np.float64(a), np.float64(b))
        assert F(float(p)) + F(float(e)) == F(a) * F(b)


def test_illcond_structure(orc):
    """A = Q orthonormal to FP64x2 accuracy; C has one 1 per column and entries
    of magnitude in (t, 10t) elsewhere; the exact A B equals C
    up to the orthogonality residual."""
    t = 1e-19
    d = G.gen_illcond(5, 48, t)
    C = d["C_target"]
    assert np.all((C == 1.0).sum(axis=0) == 1)
    off = np.abs(C[C != 1.0])
    assert np.all((off > t) & (off < 10 * t))
    n = 48
    ii, jj = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    # Q Q^T - I, exactly
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["A_hi"].T.copy(), d["A_lo"].T.copy(),
                          ii.ravel(), jj.ravel())
    assert np.max(np.abs(r["ex_hi"] - np.eye(n).ravel())) <= 2.0 ** -95
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel())
    assert np.max(np.abs(r["ex_hi"] - C.ravel())) <= 2.0 ** -95
    # most products are badly conditioned: |x^T y| ~ t while ||x|| ||y|| ~ 1
    cond = r["absab"] / np.abs(r["ex_hi"])
    assert np.median(cond) > 1e16


def test_widerange_ranges():
    """Rows of A / columns of B filled uniformly inside random ranges with
    exponents in [1e-60, 1e20]."""
    d = G.gen_widerange(7, 30, 20, 40)
    for M in (d["A_hi"], d["B_hi"].T):
        a = np.abs(M)
        assert a.min() >= 1e-60 and a.max() <= 1e20
        for row in M:  # one sign per row / column
            assert np.all(row > 0) or np.all(row < 0)
    for x in (d["A_hi"] + d["A_lo"], d["B_hi"] + d["B_lo"]):
        assert np.all(x == x)
