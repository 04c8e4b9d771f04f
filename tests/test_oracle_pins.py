"""Pins of the CPU oracle (oracle/) to things other than itself (-m "not gpu").

Each test names the PAPER.md passage (P:Lnnn) or SPEC.md example (S:Lnnn) it
pins.  Ground truth is exact rational arithmetic (fractions.Fraction), values
printed in the paper, closed-form bounds and invariants — never the oracle
re-called or its formula retyped.
"""

import math
import os
import random
import subprocess
from fractions import Fraction as F

import numpy as np
import pytest

import casc_inputs as I

W256 = (22, 21, 21)


def fr(x):
    return F(float(x))


def rnd_double(rng, lo_exp=-300, hi_exp=300):
    return rng.choice([-1, 1]) * math.ldexp(rng.random() + 0.5, rng.randint(lo_exp, hi_exp))


def rn(q: F) -> float:
    """Round a rational to the nearest double (ties to even) — Python's float(F)."""
    return float(q)


# ----------------------------------------------------------------- DD primitives
def test_two_sum_two_prod_exact(orc):
    """EFT identities s + e = a + b, p + e = a b exactly."""
    rng = random.Random(1)
    for _ in range(20000):
        a, b = rnd_double(rng, -200, 200), rnd_double(rng, -200, 200)
        s, e = orc.two_sum(a, b)
        assert s == a + b and fr(s) + fr(e) == fr(a) + fr(b)
        p, e = orc.two_prod(a, b)
        assert p == a * b and fr(p) + fr(e) == fr(a) * fr(b)


def test_spec_dd_examples(orc):
    """S:L54 two_prod(2^27+1, 2^27+1) = (2^54+2^28, 1); S:L46 two_sum(1, 2^-60)."""
    assert orc.two_prod(2.0**27 + 1, 2.0**27 + 1) == (2.0**54 + 2.0**28, 1.0)
    assert orc.two_sum(1.0, 2.0**-60) == (1.0, 2.0**-60)
    assert orc.two_sum(2.0**53, 1.0) == (2.0**53, 1.0)
    assert orc.dd_add(1.0, 0.0, -1.0, 0.0) == (0.0, 0.0)


def test_dd_add_mul_accuracy(orc):
    """dd_add / dd_mul within 2^-104 relative of the exact result."""
    rng = random.Random(2)
    for _ in range(5000):
        xh = rnd_double(rng, -100, 100)
        xl = xh * 2.0**-53 * (2 * rng.random() - 1)
        yh = rnd_double(rng, -100, 100)
        yl = yh * 2.0**-53 * (2 * rng.random() - 1)
        X, Y = fr(xh) + fr(xl), fr(yh) + fr(yl)
        h, l = orc.dd_mul(xh, xl, yh, yl)
        assert abs(fr(h) + fr(l) - X * Y) <= F(2) ** -104 * abs(X * Y)
        h, l = orc.dd_add(xh, xl, yh, yl)
        S = X + Y
        assert abs(fr(h) + fr(l) - S) <= F(2) ** -104 * (abs(X) + abs(Y))
        assert h + l == h  # normalised


# ----------------------------------------------------------------- widths a1
def test_widths_paper_values(orc):
    """(22,21,21) at k=256 ("22+21+21+53 = 117") and c0=23
    at k=64; k=1 -> (26,25,25)."""
    assert orc.select_widths(256) == (22, 21, 21)
    assert orc.select_widths(4096) == (22, 21, 21)  # k_eff = min(k, k_C), reading R3
    assert orc.select_widths(64)[0] == 23
    assert orc.select_widths(1) == (26, 25, 25)
    c = orc.select_widths(256)
    assert sum(c) + 53 == 117  # eps_tilde = 2^-117


@pytest.mark.parametrize("k", [1, 2, 3, 7, 16, 64, 100, 128, 200, 255, 256])
def test_widths_keep_bins_exact_worst_case(orc, k):
    """Brute force: with every slice at its largest magnitude on its grid
    (|s| <= 1, grid 2^(1-c), reading R4) the bin 0/1/2 sums of k terms stay
    below 2^53 grid units, i.e. FP64 accumulation of bins 0-2 is exact."""
    c0, c1, c2 = orc.select_widths(k)
    # bin0: A0 B0; grid 2^(2-2c0); |term| <= 1
    assert k * 2 ** (2 * c0 - 2) < 2**53
    # bin1 (ref sigma1): A0 B1 + A1 B0, grid 2^(2-c0-c1)
    assert 2 * k * 2 ** (c0 + c1 - 2) < 2**53
    # bin2 (ref sigma2): A0 B2 + 2^(c1-c0) A1 B1 + A2 B0, grid 2^(2-c1-max(c1,c2))
    g = 2 - c1 - max(c1, c2)
    assert (2 * k + k * 2 ** (c1 - c0)) * 2 ** (-g) < 2**53


# ----------------------------------------------------------------- exponent a2
def test_scale_exponent_invariant(orc):
    """||x||_inf <= 2^e <= 2 ||x||_inf; all-zero -> e = 0."""
    rng = np.random.default_rng(3)
    for _ in range(300):
        x = rng.standard_normal(rng.integers(1, 300)) * 2.0 ** rng.integers(-60, 60)
        if rng.random() < 0.2:
            x[rng.integers(0, x.size)] = 2.0 ** rng.integers(-20, 20)  # exact power of two
        e = orc.scale_exponent(x)
        mx = np.max(np.abs(x))
        assert mx < 2.0**e <= 2 * mx
    assert orc.scale_exponent(np.zeros(5)) == 0
    assert orc.scale_exponent(np.array([0.75, -3.5])) == 2
    assert orc.scale_exponent(np.array([1.0])) == 1


# ----------------------------------------------------------------- split a3
def test_split_spec_worked_example(orc):
    """x = (1+2^-30, 2^-70), e = 1, k = 256 -> (0.5, 2^-9, 0, 2^-7)."""
    assert orc.split_scalar(1 + 2.0**-30, 2.0**-70, 1, W256) == (0.5, 2.0**-9, 0.0, 2.0**-7)
    assert orc.split_scalar(1.0, 0.0, 1, W256) == (0.5, 0.0, 0.0, 0.0)


def _split_checks(orc, hi, lo, e, c):
    D0, D1, D2 = c[0], c[0] + c[1], c[0] + c[1] + c[2]
    sig = [F(1), F(2) ** -D0, F(2) ** -D1, F(2) ** -D2]
    s_hi = orc.split_scalar(hi, 0.0, e, c)
    s_lo = orc.split_scalar(lo, 0.0, e, c)
    chi = orc.split_scalar(hi, lo, e, c)
    # per-limb reconstruction is exact (App. A: v - s_t is exact, s_3 = remainder)
    for limb, s in ((hi, s_hi), (lo, s_lo)):
        assert sum(sg * fr(v) for sg, v in zip(sig, s)) == fr(limb) * F(2) ** -e
        for t in range(3):  # grid 2^(1-c_t), |s_t| <= 1 (reading R4)
            q = fr(s[t]) * F(2) ** (c[t] - 1)
            assert q.denominator == 1 and abs(s[t]) <= 1
    # merge: slices 0-2 exact, slice 3 = RN of the exact remainder (reading R6)
    for t in range(3):
        assert fr(chi[t]) == fr(s_hi[t]) + fr(s_lo[t])
    assert chi[3] == rn(fr(s_hi[3]) + fr(s_lo[3]))
    # eqn:error_scalar: |x 2^-e - sum sigma_t chi_t| <= 2^-(D2+53)
    X = (fr(hi) + fr(lo)) * F(2) ** -e
    err = abs(X - sum(sg * fr(v) for sg, v in zip(sig, chi)))
    assert err <= F(2) ** -(D2 + 53)
    # tail dominance: if chi0..2 = 0 the error is <= eps_mach |x|
    if chi[0] == chi[1] == chi[2] == 0:
        assert err <= F(2) ** -53 * abs(X)
    return chi


def test_split_scalar_exact_rationals(orc):
    rng = random.Random(4)
    for k in (1, 64, 256):
        c = orc.select_widths(k)
        for _ in range(3000):
            e = rng.randint(-5, 5)
            hi = rnd_double(rng, e - 40, e - 1) if rng.random() < 0.95 else 0.0
            if abs(hi) >= 2.0**e:
                hi = math.copysign(2.0**e - 2.0 ** (e - 53), hi)
            lo = hi * 2.0**-53 * (2 * rng.random() - 1)
            _split_checks(orc, hi, lo, e, c)


def test_split_full_mantissa_distribution(orc):
    """Leading zeros and slice-3 rounding (SURVEY.md §8(d) full-mantissa set)."""
    hi, lo = I.full_mantissa(7, 40, 64)
    c = orc.select_widths(256)
    for i in range(hi.shape[0]):
        e = orc.scale_exponent(hi[i])
        for p in range(hi.shape[1]):
            _split_checks(orc, hi[i, p], lo[i, p], e, c)


def test_split_panels_and_derived_b(orc):
    """Panels split conformally per row / column (§3.4);
    B4, B5, B6 are one RNE add each of exactly scaled slices (P:L1403-1404,
    reading R7); reconstruction within eqn:sigma."""
    d = I.make_config(0, m=24, n=40, k=200, seed=11)
    c = orc.select_widths(200)
    D0, D1, D2 = c[0], c[0] + c[1], c[0] + c[1] + c[2]
    SA, e = orc.split_a_panel(d["A_hi"], d["A_lo"])
    for i in range(24):
        assert e[i] == orc.scale_exponent(d["A_hi"][i])
        for p in range(0, 200, 7):
            assert tuple(SA[:, i, p]) == orc.split_scalar(d["A_hi"][i, p], d["A_lo"][i, p],
                                                         int(e[i]), c)
    SB, f = orc.split_b_panel(d["B_hi"], d["B_lo"])
    eps_t = F(2) ** -(D2 + 53)
    for j in range(40):
        assert f[j] == orc.scale_exponent(d["B_hi"][:, j])
        colmax = max(abs(fr(x)) for x in d["B_hi"][:, j])
        for p in range(200):
            b = [fr(SB[t, p, j]) for t in range(7)]
            assert SB[4, p, j] == rn(b[2] + b[3] * F(2) ** -c[2])
            assert SB[5, p, j] == rn(b[1] + b[4] * F(2) ** -c[1])
            assert SB[6, p, j] == rn(b[0] + b[5] * F(2) ** -c[0])
            rec = (b[0] + b[1] * F(2) ** -D0 + b[2] * F(2) ** -D1 + b[3] * F(2) ** -D2) \
                * F(2) ** int(f[j])
            X = fr(d["B_hi"][p, j]) + fr(d["B_lo"][p, j])
            assert abs(rec - X) <= 2 * eps_t * colmax  # eqn:sigma


# ----------------------------------------------------------------- bins a5
def _exact_bins(SA, SB, c, i, j):
    D0, D1, D2 = c[0], c[0] + c[1], c[0] + c[1] + c[2]
    a = [[fr(SA[t, i, p]) for p in range(SA.shape[2])] for t in range(4)]
    b = [[fr(SB[t, p, j]) for p in range(SB.shape[1])] for t in range(4)]
    kp = SA.shape[2]
    sig = [F(1), F(2) ** -D0, F(2) ** -D1, F(2) ** -D2]
    # sixteen-product form (eqn:Gemm16) of the reconstructed slices
    full = sum(sig[s] * sig[t] * a[s][p] * b[t][p] for s in range(4) for t in range(4)
               for p in range(kp))
    bin0 = sum(a[0][p] * b[0][p] for p in range(kp))
    bin1 = sum(a[0][p] * b[1][p] + a[1][p] * b[0][p] for p in range(kp))
    bin2 = sum(a[0][p] * b[2][p] + a[1][p] * b[1][p] * sig[1] ** 2 / sig[2] + a[2][p] * b[0][p]
               for p in range(kp))
    return full, bin0, bin1, bin2, sig


@pytest.mark.parametrize("k,seed", [(64, 0), (256, 1), (131, 2)])
def test_bins_exact_and_ten_product_identity(orc, k, seed):
    """Bins 0-2 equal their exact rational sums bit for bit ("computed
    exactly"), and bin0 + s1 bin1 + s2 bin2 + s3 bin36* reproduces the exact
    16-product sum (eqn:Gemm16 = eqn:Gemm10 with B4..B6 exact).
    The oracle's rounded bin36 is within gamma_{4k+1} sum|terms| of exact."""
    d = I.make_config(1, m=6, n=5, k=k, seed=seed)
    c = orc.select_widths(k)
    SA, _ = orc.split_a_panel(d["A_hi"], d["A_lo"])
    SB, _ = orc.split_b_panel(d["B_hi"], d["B_lo"])
    bins = orc.panel_bins(SA, SB, c)
    u = F(2) ** -53
    for i in range(6):
        for j in range(5):
            full, b0, b1, b2, sig = _exact_bins(SA, SB, c, i, j)
            assert fr(bins[0, i, j]) == b0 and fr(bins[1, i, j]) == b1
            assert fr(bins[2, i, j]) == b2
            # exact bin 3-6 with exact (unrounded) B4, B5, B6
            a = [[fr(SA[t, i, p]) for p in range(k)] for t in range(4)]
            bb = [[fr(SB[t, p, j]) for p in range(k)] for t in range(4)]
            b4 = [bb[2][p] + bb[3][p] * sig[3] / sig[2] for p in range(k)]
            b5 = [bb[1][p] + bb[2][p] * sig[2] / sig[1] + bb[3][p] * sig[3] / sig[1]
                  for p in range(k)]
            b6 = [bb[0][p] + sig[1] * bb[1][p] + sig[2] * bb[2][p] + sig[3] * bb[3][p]
                  for p in range(k)]
            s36 = sum(sig[3] * a[0][p] * bb[3][p] + sig[1] * sig[2] * a[1][p] * b4[p]
                      + sig[2] * sig[1] * a[2][p] * b5[p] + sig[3] * a[3][p] * b6[p]
                      for p in range(k))
            assert b0 + sig[1] * b1 + sig[2] * b2 + s36 == full
            # oracle bin36 (rounded slices B4..B6 and FP64 sum) vs its own exact value
            y = [[fr(SB[t, p, j]) for p in range(k)] for t in range(7)]
            f36 = sig[1] * sig[2] / sig[3]
            terms = [a[0][p] * y[3][p] for p in range(k)] + \
                [f36 * a[1][p] * y[4][p] for p in range(k)] + \
                [f36 * a[2][p] * y[5][p] for p in range(k)] + \
                [a[3][p] * y[6][p] for p in range(k)]
            ex36 = sum(terms)
            n_ops = 4 * k + 1
            gamma = n_ops * u / (1 - n_ops * u)
            assert abs(fr(bins[3, i, j]) - ex36) <= gamma * sum(abs(t) for t in terms)


def test_mutation_canary_alignment(orc, tmp_path):
    """S:L602 canary: an oracle built with a wrong in-bin alignment factor must
    fail the ten-product identity above (so that identity really pins R8)."""
    import ctypes

    import oracle
    so = str(tmp_path / "liboracle_mut.so")
    subprocess.check_call(["gcc", *oracle.CFLAGS, "-DORC_MUTATE_ALIGN", "-o", so,
                           oracle._SRC, oracle._SRC_I8, "-lm"])
    L = ctypes.CDLL(so)
    oracle._setup(L)
    d = I.make_config(1, m=3, n=3, k=64, seed=5)
    c = orc.select_widths(64)
    SA, _ = orc.split_a_panel(d["A_hi"], d["A_lo"])
    SB, _ = orc.split_b_panel(d["B_hi"], d["B_lo"])
    bins = np.empty((4, 3, 3))
    cc = (ctypes.c_int * 3)(*c)
    L.orc_panel_bins(3, 3, 64, oracle._p(SA), oracle._p(SB), cc, oracle._p(bins))
    bad = 0
    for i in range(3):
        for j in range(3):
            full, b0, b1, b2, sig = _exact_bins(SA, SB, c, i, j)
            bad += fr(bins[2, i, j]) != b2
    assert bad > 0


# ----------------------------------------------------------------- combine a6
def test_combine_closed_form(orc):
    """fl_casc = the exact weighted bin sum to DD accuracy;
    S:L433 example: bin0 = 0.5, e = f = 1 -> (2.0, 0)."""
    assert orc.combine(0.5, 0.0, 0.0, 0.0, 2, W256) == (2.0, 0.0)
    assert orc.combine(0.0, 0.0, 0.0, 0.0, 0, W256) == (0.0, 0.0)
    rng = random.Random(6)
    D0, D1, D2 = 22, 43, 64
    for _ in range(5000):
        b = [rng.randint(-2**50, 2**50) * 2.0**-44 for _ in range(3)] + [rng.uniform(-300, 300)]
        es = rng.randint(-40, 40)
        th, tl = orc.combine(*b, es, W256)
        ex = (fr(b[0]) + fr(b[1]) * F(2) ** -D0 + fr(b[2]) * F(2) ** -D1
              + fr(b[3]) * F(2) ** -D2) * F(2) ** es
        assert abs(fr(th) + fr(tl) - ex) <= F(2) ** -104 * abs(ex) + F(2) ** (-1000)
        assert th + tl == th


# ----------------------------------------------------------------- final C
def _check_vs_exact(orc, d, C_hi, C_lo, nthreads=0):
    m, n, k = d["m"], d["n"], d["k"]
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo, nthreads=nthreads)
    ratio = np.abs(r["err"]) / np.maximum(orc.north_star_bound(k, r["absab"]), 1e-300)
    return ratio.max(), r


@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 37, 29, 600), (2, 48, 40, 513),
                                       (1, 1, 1, 1), (1, 5, 3, 257)])
def test_cascade_within_north_star_bound(orc, cfg, m, n, k):
    """Final C within 4 k 2^-104 |A||B| of the exact product (BASELINE north
    star), on every entry; k > 256 covers the FP64x2 cross-panel accumulation
    (P:L2839)."""
    d = I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, flags = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    worst, _ = _check_vs_exact(orc, d, C_hi, C_lo)
    assert worst <= 1.0
    assert flags.sum() == 0  # uniform data: bin 0 never vanishes
    assert np.all(C_hi + C_lo == C_hi)


def test_dd_gemm_within_bound(orc):
    """ORACLE-DD within its FP64x2 bound gamma_k |A||B| (eqn:fp64x2,
    P:L2891-2897), taken generously as 4 k 2^-104."""
    d = I.make_config(1, m=20, n=21, k=300)
    C_hi, C_lo = orc.dd_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    worst, _ = _check_vs_exact(orc, d, C_hi, C_lo)
    assert worst <= 1.0


def test_worst_case_example_flagged(orc):
    """§3.6 worst case x = (1, eps), y = (0, 1): cascaded result
    is fl64(eps) and bin 0 vanishes -> flagged; S:L379 eps = 2^-100 -> exact."""
    for eps in (2.0**-100, 2.0**-70 * 1.2345, 3e-25):
        A_hi = np.array([[1.0, eps]])
        A_lo = np.zeros((1, 2))
        B_hi = np.array([[0.0], [1.0]])
        B_lo = np.zeros((2, 1))
        C_hi, C_lo, flags = orc.casc_gemm(A_hi, A_lo, B_hi, B_lo)
        assert flags[0, 0] == 1
        assert abs(C_hi[0, 0] + C_lo[0, 0] - eps) <= 2.0**-52 * eps
    C_hi, C_lo, flags = orc.casc_gemm(np.array([[1.0, 2.0**-100]]), np.zeros((1, 2)),
                                      np.array([[0.0], [1.0]]), np.zeros((2, 1)))
    assert (C_hi[0, 0], C_lo[0, 0]) == (2.0**-100, 0.0)


def test_identity_and_zero_rows(orc):
    """A = I -> C = B within 2^-116 column max; zero rows of A give
    zero rows of C, flagged (bin 0 == 0)."""
    d = I.make_config(1, m=40, n=17, k=40, seed=9)
    A_hi = np.eye(40)
    A_hi[7] = 0.0
    C_hi, C_lo, flags = orc.casc_gemm(A_hi, np.zeros((40, 40)), d["B_hi"], d["B_lo"])
    for i in range(40):
        for j in range(17):
            if i == 7:
                assert C_hi[i, j] == 0 and C_lo[i, j] == 0 and flags[i, j] == 1
                continue
            colmax = np.max(np.abs(d["B_hi"][:, j]))
            err = abs(fr(C_hi[i, j]) + fr(C_lo[i, j]) - fr(d["B_hi"][i, j]) - fr(d["B_lo"][i, j]))
            assert err <= F(2) ** -116 * fr(colmax)


def test_scaling_neutrality(orc):
    """Scaling row i of A by 2^u_i and column j of B by 2^v_j scales C exactly
    (the per-row/column Sigma, T of §3.4): bitwise."""
    d = I.make_config(1, m=30, n=20, k=300, seed=3)
    s = I.make_config(2, m=30, n=20, k=300, seed=3)
    C0 = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    C1 = orc.casc_gemm(s["A_hi"], s["A_lo"], s["B_hi"], s["B_lo"])
    u = I.int_uniform(3, I.STREAM_ROW_EXP, 30, -30, 30)
    v = I.int_uniform(3, I.STREAM_COL_EXP, 20, -30, 30)
    sc = np.ldexp(1.0, (u[:, None] + v[None, :]))
    assert np.array_equal(C0[0] * sc, C1[0]) and np.array_equal(C0[1] * sc, C1[1])
    assert np.array_equal(C0[2], C1[2])


def test_cancellation_variants(orc):
    """cfg3 structure at small size (reading R13): 3a literal column negation
    creates no in-dot-product cancellation (no flags); 3b in-panel pairing
    flags every entry; 3c cross-panel pairing is invisible to the per-panel
    detector ("where k <= k_C"). All stay within the north-star bound
    except where flagged."""
    for variant, expect in (("a", "none"), ("b", "all"), ("c", "none")):
        d = I.make_config(3, m=12, n=10, k=1024, variant=variant)
        C_hi, C_lo, flags = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
        if expect == "none":
            assert flags.sum() == 0
            worst, _ = _check_vs_exact(orc, d, C_hi, C_lo)
            assert worst <= 1.0
        else:
            assert flags.all()


def test_blas_ex_oracle(orc):
    """NEXT-4 oracle: alpha = 1, beta = 0 is the plain product (bitwise); op(X)
    = X^T is pure data movement (bitwise); alpha = 2^p scales exactly; general
    alpha, beta within the FP64x2 update bound of the exact alpha AB + beta C."""
    d = I.make_config(1, m=9, n=7, k=300, seed=17)
    P = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    C0 = (np.zeros((9, 7)), np.zeros((9, 7)))
    E = orc.casc_gemm_ex("N", "N", (1.0, 0.0), d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"],
                         (0.0, 0.0), *C0)
    assert np.array_equal(E[0], P[0]) and np.array_equal(E[1], P[1]) and np.array_equal(E[2], P[2])
    T = orc.casc_gemm_ex("T", "T", (1.0, 0.0), d["A_hi"].T.copy(), d["A_lo"].T.copy(),
                         d["B_hi"].T.copy(), d["B_lo"].T.copy(), (0.0, 0.0), *C0)
    assert np.array_equal(T[0], P[0]) and np.array_equal(T[1], P[1])
    S = orc.casc_gemm_ex("N", "N", (0.25, 0.0), d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"],
                         (0.0, 0.0), *C0)
    assert np.array_equal(S[0], P[0] * 0.25) and np.array_equal(S[1], P[1] * 0.25)
    rng = np.random.default_rng(4)
    Ch, Cl = rng.uniform(-1, 1, (9, 7)), np.zeros((9, 7))
    al, be = (1.0 / 3.0, 1.0 / 3.0 * 2.0 ** -54), (-0.7, 2.0 ** -60)
    G = orc.casc_gemm_ex("N", "N", al, d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], be, Ch, Cl)
    for i in range(9):
        for j in range(7):
            ab = sum((fr(d["A_hi"][i, p]) + fr(d["A_lo"][i, p]))
                     * (fr(d["B_hi"][p, j]) + fr(d["B_lo"][p, j])) for p in range(300))
            absab = sum(abs(fr(d["A_hi"][i, p]) + fr(d["A_lo"][i, p]))
                        * abs(fr(d["B_hi"][p, j]) + fr(d["B_lo"][p, j])) for p in range(300))
            A_ = fr(al[0]) + fr(al[1])
            B_ = fr(be[0]) + fr(be[1])
            ex = A_ * ab + B_ * fr(Ch[i, j])
            bound = abs(A_) * 4 * 300 * F(2) ** -104 * absab + F(2) ** -102 * (
                abs(A_ * ab) + abs(B_ * fr(Ch[i, j])))
            assert abs(fr(G[0][i, j]) + fr(G[1][i, j]) - ex) <= bound
    Z = orc.casc_gemm_ex("N", "N", (0.0, 0.0), d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], be,
                         Ch, Cl)  # alpha = 0: C := beta C
    for i in range(9):
        for j in range(7):
            assert abs(fr(Z[0][i, j]) + fr(Z[1][i, j]) - (fr(be[0]) + fr(be[1])) * fr(Ch[i, j])) \
                <= F(2) ** -104 * abs(fr(Ch[i, j]))
    assert Z[2].sum() == 0


@pytest.mark.parametrize("uplo,trans", [("L", "N"), ("U", "N"), ("L", "T"), ("U", "T")])
def test_syrk_oracle(orc, uplo, trans):
    """NEXT-4 SYRK oracle: on its triangle, alpha = 1, beta = 0 is within
    the north-star bound of the exact op(A) op(A)^T (exact rationals); the other
    triangle and its flags are untouched; alpha = 2^p scales exactly; beta = 0
    does not read C; alpha = 0 scales the triangle by beta."""
    n, k = 11, 300
    d = I.make_config(1, m=n, n=k, k=k, seed=19)
    A_hi, A_lo = d["A_hi"][:n, :k], d["A_lo"][:n, :k]  # op(A): n x k
    Ast = (A_hi.T.copy(), A_lo.T.copy()) if trans == "T" else (A_hi.copy(), A_lo.copy())
    sent = np.full((n, n), 7.5)
    fl0 = np.full((n, n), 9, np.uint8)
    Ch, Cl, fl = orc.casc_syrk(uplo, trans, (1.0, 0.0), *Ast, (0.0, 0.0), sent, sent, fl0)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    assert np.all(Ch[~tri] == 7.5) and np.all(Cl[~tri] == 7.5) and np.all(fl[~tri] == 9)
    assert np.all(fl[tri] <= 1)
    for i in range(n):
        for j in range(n):
            if not tri[i, j]:
                continue
            ex = sum((fr(A_hi[i, p]) + fr(A_lo[i, p])) * (fr(A_hi[j, p]) + fr(A_lo[j, p]))
                     for p in range(k))
            absab = sum(abs(fr(A_hi[i, p]) + fr(A_lo[i, p])) * abs(fr(A_hi[j, p]) + fr(A_lo[j, p]))
                        for p in range(k))
            assert abs(fr(Ch[i, j]) + fr(Cl[i, j]) - ex) <= 4 * k * F(2) ** -104 * absab
    S = orc.casc_syrk(uplo, trans, (8.0, 0.0), *Ast, (0.0, 0.0), sent, sent)
    assert np.array_equal(S[0][tri], 8 * Ch[tri]) and np.array_equal(S[1][tri], 8 * Cl[tri])
    nan = np.full((n, n), np.nan)
    N_ = orc.casc_syrk(uplo, trans, (1.0, 0.0), *Ast, (0.0, 0.0), nan, nan)
    assert np.array_equal(N_[0][tri], Ch[tri]) and np.all(np.isnan(N_[0][~tri]))
    rng = np.random.default_rng(8)
    C0 = rng.uniform(-1, 1, (n, n))
    Z = orc.casc_syrk(uplo, trans, (0.0, 0.0), *Ast, (0.5, 0.0), C0, np.zeros((n, n)), fl0)
    assert np.array_equal(Z[0][tri], 0.5 * C0[tri]) and np.array_equal(Z[0][~tri], C0[~tri])
    assert np.all(Z[2][tri] == 0) and np.all(Z[2][~tri] == 9)


def _tri_dd(m, uplo, seed, unit=False):
    """Diagonally dominant triangular FP64x2 matrix (well conditioned)."""
    rng = np.random.default_rng(seed)
    hi = rng.uniform(-1, 1, (m, m)) / m
    hi = np.tril(hi) if uplo == "L" else np.triu(hi)
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, (m, m))
    d = 1.0 + rng.uniform(0, 1, m)
    hi[np.arange(m), np.arange(m)] = 1.0 if unit else d
    lo[np.arange(m), np.arange(m)] = 0.0 if unit else d * 2.0 ** -54
    return hi, lo


def test_dd_div_oracle(orc):
    """R27 FP64x2 division: within 2^-100 of the exact quotient (Fractions)."""
    rng = random.Random(5)
    for _ in range(3000):
        xh = rng.uniform(-1, 1) * 2.0 ** rng.randint(-40, 40)
        yh = rng.uniform(0.5, 1) * (-1) ** rng.randint(0, 1) * 2.0 ** rng.randint(-40, 40)
        xl = xh * 2.0 ** -53 * rng.uniform(-1, 1)
        yl = yh * 2.0 ** -53 * rng.uniform(-1, 1)
        qh, ql = orc.dd_div(xh, xl, yh, yl)
        ex = (fr(xh) + fr(xl)) / (fr(yh) + fr(yl))
        assert abs(fr(qh) + fr(ql) - ex) <= abs(ex) * F(2) ** -100
        assert abs(ql) <= abs(qh) * 2.0 ** -52  # normalised


@pytest.mark.parametrize("uplo,unit", [("L", False), ("U", False), ("L", True)])
def test_trsm_diag_inverse_oracle(orc, uplo, unit):
    """R27 diagonal-block inverses: Inv_b A_bb = I within 2^-95 (exact rationals),
    zeros outside the triangle, the ragged last block included."""
    m = 300
    A_hi, A_lo = _tri_dd(m, uplo, 3, unit)
    Ih, Il = orc.trsm_diag_inv(uplo, "U" if unit else "N", A_hi, A_lo)
    assert Ih.shape == (2, 256, 256)
    for b, (r0, nb, cols) in enumerate([(0, 256, (0, 97, 255)), (256, 44, range(44))]):
        inv = Ih[b][:nb, :nb]
        tri = np.tril(np.ones((nb, nb), bool)) if uplo == "L" else np.triu(np.ones((nb, nb), bool))
        assert np.all(inv[~tri] == 0) and np.all(Ih[b][nb:, :] == 0)
        for j in cols:
            for i in range(0, nb, 7 if nb > 64 else 1):
                s = sum((fr(Ih[b][i, l]) + fr(Il[b][i, l]))
                        * (fr(A_hi[r0 + l, r0 + j]) + fr(A_lo[r0 + l, r0 + j])) for l in range(nb))
                assert abs(s - (1 if i == j else 0)) <= F(2) ** -95


@pytest.mark.parametrize("uplo,trans,unit,m,n", [("L", "N", False, 40, 5), ("U", "N", False, 300, 3),
                                                 ("L", "N", True, 300, 2), ("L", "T", False, 300, 2),
                                                 ("U", "T", False, 40, 3), ("L", "N", False, 1100, 1),
                                                 ("U", "T", False, 1100, 1)])
def test_trsm_oracle(orc, uplo, trans, unit, m, n):
    """R27 TRSM: the exact residual of op(A) X = B (dyadic rationals, no
    rounding) within 2^-96 (|op(A)||X|) row by row (diagonally dominant A, so
    X is then accurate; two blocks with the cascaded-GEMM update for m = 300)
    and, for m = 40, X within 2^-95 of the exact solution; alpha = 2 scales
    exactly; alpha = 0 gives X = 0."""
    A_hi, A_lo = _tri_dd(m, uplo, 7, unit)
    rng = np.random.default_rng(9)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))  # normalised pairs: exact scaling
    X_hi, X_lo = orc.casc_trsm(uplo, "U" if unit else "N", (1.0, 0.0), A_hi, A_lo, B_hi, B_lo,
                               trans=trans)
    A = [[fr(A_hi[i, j]) + fr(A_lo[i, j]) for j in range(m)] for i in range(m)]
    if trans == "T":
        A = [list(r) for r in zip(*A)]  # op(A)
    lower = (uplo == "L") != (trans == "T")
    X = [[fr(X_hi[i, j]) + fr(X_lo[i, j]) for j in range(n)] for i in range(m)]
    for i in range(0, m, 1 if m <= 40 else (9 if m <= 300 else 97)):
        lo, hi = (0, i + 1) if lower else (i, m)
        for j in range(n):
            r = sum(A[i][l] * X[l][j] for l in range(lo, hi)) - (fr(B_hi[i, j]) + fr(B_lo[i, j]))
            mag = sum(abs(A[i][l] * X[l][j]) for l in range(lo, hi))
            assert abs(r) <= F(2) ** -96 * mag
    if m <= 40:  # exact solution by substitution
        order = range(m) if lower else range(m - 1, -1, -1)
        for j in range(n):
            x = [F(0)] * m
            for i in order:
                lo, hi = (0, i) if lower else (i + 1, m)
                x[i] = (fr(B_hi[i, j]) + fr(B_lo[i, j])
                        - sum(A[i][l] * x[l] for l in range(lo, hi))) / A[i][i]
            for i in range(m):
                assert abs(X[i][j] - x[i]) <= F(2) ** -95 * (abs(x[i]) + 1)
    Y = orc.casc_trsm(uplo, "U" if unit else "N", (2.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    assert np.array_equal(Y[0], 2 * X_hi) and np.array_equal(Y[1], 2 * X_lo)
    Z = orc.casc_trsm(uplo, "N", (0.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    assert np.all(Z[0] == 0) and np.all(Z[1] == 0)


def test_exact_accumulator_vs_fractions(orc):
    """ORACLE-EXACT superaccumulator equals Fraction sums, over
    wide exponent ranges and with exact cancellation."""
    rng = random.Random(8)
    for trial in range(200):
        n = rng.randint(1, 60)
        x = [rnd_double(rng, -600, 600) for _ in range(n)]
        y = [rnd_double(rng, -400, 400) for _ in range(n)]
        if trial % 5 == 0:
            x += [-v for v in x]
            y += y
        h, l = orc.exact_dot(np.array(x), np.array(y))
        ex = sum(fr(a) * fr(b) for a, b in zip(x, y))
        assert h == rn(ex)
        assert l == rn(ex - fr(h))
        h, l = orc.exact_sum(np.array(x))
        ex = sum(fr(a) for a in x)
        assert h == rn(ex) and l == rn(ex - fr(h))


def test_exact_entries_vs_fractions(orc):
    d = I.make_config(2, m=4, n=3, k=50, seed=12)
    ii, jj = np.meshgrid(np.arange(4), np.arange(3), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel())
    for t, (i, j) in enumerate(zip(ii.ravel(), jj.ravel())):
        ex = sum((fr(d["A_hi"][i, p]) + fr(d["A_lo"][i, p]))
                 * (fr(d["B_hi"][p, j]) + fr(d["B_lo"][p, j])) for p in range(50))
        ab = sum(abs(fr(d["A_hi"][i, p]) + fr(d["A_lo"][i, p]))
                 * abs(fr(d["B_hi"][p, j]) + fr(d["B_lo"][p, j])) for p in range(50))
        assert r["ex_hi"][t] == rn(ex) and r["ex_lo"][t] == rn(ex - fr(r["ex_hi"][t]))
        assert r["absab"][t] == rn(ab)


def test_inputs_normalised_and_blockwise():
    """Generator: (hi, lo) normalised (|lo| <= ulp(hi)/2) and any row block is
    bit-identical to the same rows of the full matrix (P-invariance premise)."""
    d = I.make_config(4, m=64, n=48, k=80)
    assert np.all(d["A_hi"] + d["A_lo"] == d["A_hi"])
    assert np.all(d["B_hi"] + d["B_lo"] == d["B_hi"])
    blk = I.make_config(4, m=64, n=48, k=80, rows=slice(16, 40))
    assert np.array_equal(blk["A_hi"], d["A_hi"][16:40])
    assert np.array_equal(blk["A_lo"], d["A_lo"][16:40])
    assert np.abs(d["A_hi"]).max() <= 1.0
    for v in ("a", "b", "c"):  # cfg3's perturbed pairs are renormalised too (R15)
        c3 = I.make_config(3, m=8, n=64, k=1024, variant=v)
        assert np.all(c3["B_hi"] + c3["B_lo"] == c3["B_hi"])
        assert np.all(c3["A_hi"] + c3["A_lo"] == c3["A_hi"])
    for cfg in (1, 2, 3, 4):  # column slabs of B (the multi-GPU slab generation)
        kw = dict(m=12, n=200, k=300)
        f = I.make_config(cfg, **kw)
        s = I.make_config(cfg, cols=slice(64, 150), **kw)
        assert np.array_equal(f["B_hi"][:, 64:150], s["B_hi"])
        assert np.array_equal(f["B_lo"][:, 64:150], s["B_lo"])
