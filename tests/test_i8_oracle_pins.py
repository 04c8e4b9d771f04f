"""Pins of the INT8-cascade oracle (NEXT-3; oracle/casc_i8_oracle.c) to things
other than itself (-m "not gpu").

The paper sketches the variant in §6: the FP64x2 matrices are
converted to fixed point, cascaded into ~14-15 INT8 splits and multiplied with
the y(y+1)/2 INT8 products of the triangle i + j < y, accumulating in 32-bit
integers.  DESIGN.md readings R22-R26 fix the details; each test names the one
it pins.  Ground truth is exact rational arithmetic (fractions.Fraction),
hand-derived digit strings, closed-form bounds and invariants, and ORACLE-EXACT
(the superaccumulator, pinned in test_oracle_pins.py) — never the oracle's own
formula retyped.
"""

import math
import random
from fractions import Fraction as F

import numpy as np
import pytest

import casc_inputs as I


def fr(x):
    return F(float(x))


def fxpt(hi, lo, e, y):
    """X of reading R23 from its definition: each limb scaled by 2^(F-e) and
    rounded to the nearest integer, ties to even (Python's round(Fraction))."""
    Fb = 6 + 8 * (y - 1)
    s = F(2) ** (Fb - int(e))
    return round(fr(hi) * s) + round(fr(lo) * s), Fb


def digits_value(d):
    v = 0
    for t in d:
        v = v * 256 + t
    return v


# ----------------------------------------------------------------- slices (R23)
def test_i8_split_hand_examples(orc):
    """Hand-derived digit strings: 0.75 = 48 * 2^-6; -0.75; the last digit is
    2^-(6+8(y-1)); 1 - 2^-53 = 64 * 2^-6 - 2 * 2^-(6+8*6) (balanced carry)."""
    z = [0] * 13
    assert orc.i8_split_scalar(0.75, 0.0, 0, 14) == tuple([48] + z)
    assert orc.i8_split_scalar(-0.75, 0.0, 0, 14) == tuple([-48] + z)
    assert orc.i8_split_scalar(2.0**-110, 0.0, 0, 14) == tuple([0] * 13 + [1])
    assert orc.i8_split_scalar(1.5 * 2.0**-110, 0.0, 0, 14) == tuple([0] * 13 + [2])  # tie -> even
    d = [64, 0, 0, 0, 0, 0, -2] + [0] * 7
    assert orc.i8_split_scalar(1.0 - 2.0**-53, 0.0, 0, 14) == tuple(d)
    # scale exponent shifts the grid: x = 3 with e = 2 is 0.75 of the scale
    assert orc.i8_split_scalar(3.0, 0.0, 2, 5) == (48, 0, 0, 0, 0)
    # a digit of exactly -128 (byte 0x80) stays -128, it does not carry
    assert orc.i8_split_scalar(-128 * 2.0**-14, 0.0, 0, 3) == (0, -128, 0)
    assert orc.i8_split_scalar(128 * 2.0**-14, 0.0, 0, 3) == (1, -128, 0)


@pytest.mark.parametrize("y", [3, 8, 14, 15])
def test_i8_split_scalar_exact_rationals(orc, y):
    """Digits of random FP64x2 values (uniform, full-mantissa with up to 100
    leading zeros, random scale exponents at and above the value's own) sum to
    the exactly rounded fixed-point integer X of reading R23, lie in the
    balanced ranges, and X 2^-F is within 2^-F of x 2^-e."""
    rng = random.Random(100 + y)
    for it in range(3000):
        hi = rng.choice([-1, 1]) * math.ldexp(rng.random() + 0.5, -rng.randint(0, 100))
        lo = hi * 2.0**-53 * (2 * rng.random() - 1)
        hi, lo = hi + lo, lo - ((hi + lo) - hi)  # Fast2Sum renormalisation
        e = math.frexp(hi)[1] + (0 if it % 3 else rng.randint(0, 20))
        d = orc.i8_split_scalar(hi, lo, e, y)
        X, Fb = fxpt(hi, lo, e, y)
        assert digits_value(d) == X
        assert -64 <= d[0] <= 64 and all(-128 <= t <= 127 for t in d[1:])
        assert abs(F(X, 2**Fb) - (fr(hi) + fr(lo)) / F(2) ** int(e)) <= F(1, 2**Fb)


def test_i8_split_panels(orc):
    """Per-row (A) / per-column (B) scale exponents obey ||x|| < 2^e <= 2||x||
    (reading R1 applied per R22 panel) and every element's digits are
    its scalar split under that exponent."""
    d = I.make_config(2, m=6, n=5, k=70, seed=4)
    hm, lm = I.full_mantissa(5, 6, 70)
    for A_hi, A_lo in ((d["A_hi"], d["A_lo"]), (hm, lm)):
        D, e = orc.i8_split_a_panel(A_hi, A_lo, 14)
        for i in range(A_hi.shape[0]):
            mx = np.max(np.abs(A_hi[i]))
            assert mx < 2.0 ** e[i] <= 2 * mx
            for p in range(0, 70, 7):
                assert tuple(D[:, i, p]) == orc.i8_split_scalar(A_hi[i, p], A_lo[i, p], e[i], 14)
    D, f = orc.i8_split_b_panel(d["B_hi"], d["B_lo"], 14)
    for j in range(5):
        mx = np.max(np.abs(d["B_hi"][:, j]))
        assert mx < 2.0 ** f[j] <= 2 * mx
        for p in range(0, 70, 9):
            assert tuple(D[:, j, p]) == orc.i8_split_scalar(d["B_hi"][p, j], d["B_lo"][p, j],
                                                            f[j], 14)


# ----------------------------------------------------------------- bins (R24)
@pytest.mark.parametrize("y,kp", [(14, 37), (5, 64), (15, 20)])
def test_i8_all_products_equal_exact_product(orc, y, kp):
    """With every product kept (2y-1 diagonals), sum_s bin_s 2^(-12-8s) is the
    exact product of the reconstructed fixed-point values X_A 2^-F and X_B 2^-F
    (Fraction arithmetic); the paper's triangle is its first y bins
    and the dropped diagonals are bounded by sum_(s>=y) (s+1) kp 2^(14-12-8s)."""
    d = I.make_config(1, m=4, n=3, k=kp, seed=y)
    DA, e = orc.i8_split_a_panel(d["A_hi"], d["A_lo"], y)
    DB, f = orc.i8_split_b_panel(d["B_hi"], d["B_lo"], y)
    full = orc.i8_panel_bins(DA, DB, 2 * y - 1)
    tri = orc.i8_panel_bins(DA, DB)
    assert np.array_equal(full[:y], tri)
    for i in range(4):
        for j in range(3):
            exact = F(0)
            for p in range(kp):
                xa, Fb = fxpt(d["A_hi"][i, p], d["A_lo"][i, p], e[i], y)
                xb, _ = fxpt(d["B_hi"][p, j], d["B_lo"][p, j], f[j], y)
                exact += F(xa * xb, 2 ** (2 * Fb))
            got = sum(F(int(full[s, i, j])) * F(1, 2 ** (12 + 8 * s)) for s in range(2 * y - 1))
            assert got == exact
            dropped = sum(F(int(full[s, i, j])) * F(1, 2 ** (12 + 8 * s))
                          for s in range(y, 2 * y - 1))
            bound = sum(F((s + 1) * kp * 2**14, 2 ** (12 + 8 * s)) for s in range(y, 2 * y - 1))
            assert abs(dropped) <= bound


def test_i8_bins_fit_int32_worst_case(orc):
    """Reading R22: at the panel depth 8192 and y = 15 the largest possible
    bin (every digit -128 against -128; top digits 64) stays below 2^31 —
    brute force on the worst-case operands, and the closed form."""
    y, kp = 15, orc.i8_panel()
    assert kp == 8192 and y * kp * 2**14 < 2**31
    # every lower digit -128 and the top digit -64 (reachable digit values, R23)
    d = [-64] + [-128] * (y - 1)
    DA = np.array(d, dtype=np.int8)[:, None, None] * np.ones((1, 1, kp), dtype=np.int8)
    bins = orc.i8_panel_bins(DA, DA)
    for s in range(y):
        expect = sum(d[a] * d[s - a] for a in range(s + 1)) * kp
        assert bins[s, 0, 0] == expect and abs(expect) < 2**31


def test_i8_group_value_exact(orc):
    """Reading R25: the group value is exact as FP64x2 and normalised
    (hi = RN(V), lo = V - hi)."""
    rng = random.Random(7)
    for _ in range(2000):
        nb = rng.randint(1, 4)
        b = [rng.randint(-2**31 + 1, 2**31 - 1) for _ in range(nb)]
        V = digits_value(b)
        h, l = orc.i8_group_value(np.array(b))
        assert fr(h) + fr(l) == V and h == float(F(V))


def _rn_pair_expected(bins, w0):
    """T by exact rationals: hi = RN(x), lo = RN(x - hi) (Python's int / int is
    correctly rounded, ties to even, subnormals included)."""
    y = len(bins)
    S = sum(int(b) << (8 * (y - 1 - s)) for s, b in enumerate(bins))
    x = F(S) * F(2) ** w0
    hi = float(x) if S else 0.0
    r = x - F(hi)
    lo = float(r) if r else 0.0
    return hi, lo


def _bits(v):
    return np.float64(v).view(np.uint64)


def test_i8_panel_value_exact_rounding(orc):
    """Reading R25 (rev. 2): T.hi = RN(x), T.lo = RN(x - T.hi) for the exact panel
    product x, against exact rationals: random bins, ties both ways, exact zeros,
    cancelling bins and the subnormal range (bitwise, signed zeros included)."""
    rng = random.Random(11)
    cases = []
    for _ in range(3000):
        y = rng.randint(3, 15)
        b = [rng.randint(-2**31 + 1, 2**31 - 1) for _ in range(y)]
        for s in range(y):  # sparse / short / signed-mixed patterns
            if rng.random() < 0.3:
                b[s] = 0
        cases.append((b, rng.randint(-300, 200)))
    for _ in range(500):  # the subnormal range of hi and lo
        y = rng.randint(3, 15)
        b = [rng.randint(-2**31 + 1, 2**31 - 1) for _ in range(y)]
        cases.append((b, rng.randint(-1250, -1000)))
    for k in (3, 17, 40):  # ties: x = (q + 1/2) 2^k with q even and odd
        for q in (2**53 - 2, 2**53 - 1, 2**52 + 1, 2**52 + 6):
            S = (2 * q + 1) << (k - 1)
            y = 15
            digits = [(S >> (8 * (y - 1 - s))) & 0xff for s in range(y)]
            assert sum(d << (8 * (y - 1 - s)) for s, d in enumerate(digits)) == S
            cases += [(digits, 0), ([-d for d in digits], -7), (digits, -1074 - k - 20)]
    cases += [([0] * 14, 0), ([1, -256] + [0] * 12, 5), ([0] * 13 + [1], -1080),
              ([0] * 13 + [-1], -1080), ([0] * 13 + [-3], -1076)]
    for b, w0 in cases:
        h, l = orc.i8_panel_value(np.array(b), w0)
        eh, el = _rn_pair_expected(b, w0)
        assert _bits(h) == _bits(eh) and _bits(l) == _bits(el), (b, w0, h, l, eh, el)


# ----------------------------------------------------------------- final C
def _check_vs_exact(orc, d, C_hi, C_lo):
    m, n, k = d["m"], d["n"], d["k"]
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo)
    ratio = np.abs(r["err"]) / np.maximum(orc.north_star_bound(k, r["absab"]), 1e-300)
    return ratio.max()


@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 19, 23, 600), (2, 16, 12, 513),
                                       (1, 1, 1, 1), (1, 3, 4, 8192 + 300)])
def test_i8_cascade_within_north_star_bound(orc, cfg, m, n, k):
    """Final C of the y = 14 INT8 cascade (105 products) within
    4 k 2^-104 |A||B| of the exact product on every entry, including two k
    panels (k > 8192, FP64x2 cross-panel accumulation) and 1x1x1; no flags on
    uniform data."""
    d = I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, flags = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert _check_vs_exact(orc, d, C_hi, C_lo) <= 1.0
    assert flags.sum() == 0
    assert np.all(C_hi + C_lo == C_hi)


def test_i8_accuracy_grows_with_slices(orc):
    """Fewer slices lose bits: the error with y = 8 (~6 + 56 bits) is far above
    y = 14's, and y = 8 stays within 2^-60 |A||B| k."""
    d = I.make_config(1, m=8, n=8, k=200, seed=11)
    ii, jj = np.meshgrid(np.arange(8), np.arange(8), indexing="ij")
    errs = {}
    for y in (8, 14):
        C_hi, C_lo, _ = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], y)
        r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                              C_hi, C_lo)
        errs[y] = np.max(np.abs(r["err"]) / r["absab"])
    assert errs[8] <= 200 * 2.0**-60 and errs[14] < errs[8] * 2.0**-30


def test_i8_scaling_neutrality(orc):
    """Scaling row i of A by 2^u_i and column j of B by 2^v_j scales C exactly
    (per-row/column exponents, R22): bitwise, flags equal."""
    d = I.make_config(1, m=12, n=10, k=300, seed=3)
    s = I.make_config(2, m=12, n=10, k=300, seed=3)
    C0 = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    C1 = orc.i8_casc_gemm(s["A_hi"], s["A_lo"], s["B_hi"], s["B_lo"])
    u = I.int_uniform(3, I.STREAM_ROW_EXP, 12, -30, 30)
    v = I.int_uniform(3, I.STREAM_COL_EXP, 10, -30, 30)
    sc = np.ldexp(1.0, (u[:, None] + v[None, :]))
    assert np.array_equal(C0[0] * sc, C1[0]) and np.array_equal(C0[1] * sc, C1[1])
    assert np.array_equal(C0[2], C1[2])


def test_i8_identity_zero_rows_and_worst_case(orc):
    """A = I gives C = B within 4 k 2^-104 |b|; a zero row of A gives a zero row
    of C, flagged (R26); the §3.6 worst case x = (1, eps), y = (0, 1)
    is flagged."""
    d = I.make_config(1, m=20, n=9, k=20, seed=9)
    A_hi = np.eye(20)
    A_hi[7] = 0.0
    C_hi, C_lo, flags = orc.i8_casc_gemm(A_hi, np.zeros((20, 20)), d["B_hi"], d["B_lo"])
    assert np.all(C_hi[7] == 0) and np.all(C_lo[7] == 0) and np.all(flags[7] == 1)
    rows = [i for i in range(20) if i != 7]
    for i in rows:
        for j in range(9):
            err = abs(fr(C_hi[i, j]) + fr(C_lo[i, j]) - fr(d["B_hi"][i, j]) - fr(d["B_lo"][i, j]))
            assert err <= F(4 * 20, 2**104) * (abs(fr(d["B_hi"][i, j])) + F(1, 2**200))
    assert flags[rows].sum() == 0
    for eps in (2.0**-100, 2.0**-70 * 1.2345):
        C_hi, C_lo, flags = orc.i8_casc_gemm(np.array([[1.0, eps]]), np.zeros((1, 2)),
                                             np.array([[0.0], [1.0]]), np.zeros((2, 1)))
        assert flags[0, 0] == 1


def test_i8_cancellation_variants(orc):
    """cfg3 structure at small size (reading R13 with the INT8 panel of R22):
    3a literal column negation: no flags, within the bound; 3b (pairs 128
    apart) and 3c (pairs 256 apart) both cancel inside one 8192-deep panel to
    ~2^-60 of the operand scale, so every entry is flagged (R26)."""
    for variant, expect in (("a", "none"), ("b", "all"), ("c", "all")):
        d = I.make_config(3, m=8, n=6, k=1024, variant=variant)
        C_hi, C_lo, flags = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
        if expect == "none":
            assert flags.sum() == 0
            assert _check_vs_exact(orc, d, C_hi, C_lo) <= 1.0
        else:
            assert flags.all()


def test_i8_k_zero(orc):
    """k == 0: C := 0, flags := 0 (reading R18)."""
    C_hi, C_lo, flags = orc.i8_casc_gemm(np.zeros((3, 0)), np.zeros((3, 0)), np.zeros((0, 2)),
                                         np.zeros((0, 2)))
    assert np.all(C_hi == 0) and np.all(C_lo == 0) and np.all(flags == 0)


def test_i8_blas_ex_oracle(orc):
    """NEXT-4 on the INT8 cascade (reading R21): transposed storage gives the
    plain product bit for bit; alpha = 2^p scales exactly; alpha = 1, beta = 1
    adds C within 2^-104 (exact rationals); k == 0 and alpha == 0 give
    beta (x) C with no flags; beta == 0 never reads C (NaN C stays unread)."""
    d = I.make_config(1, m=9, n=7, k=300, seed=41)
    P = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    nanC = np.full((9, 7), np.nan)
    r = orc.i8_casc_gemm_ex("T", "T", (1.0, 0.0), d["A_hi"].T, d["A_lo"].T, d["B_hi"].T,
                            d["B_lo"].T, (0.0, 0.0), nanC, nanC)
    assert all(np.array_equal(x, z) for x, z in zip(r, P))
    r = orc.i8_casc_gemm_ex("N", "T", (2.0**-5, 0.0), d["A_hi"], d["A_lo"], d["B_hi"].T,
                            d["B_lo"].T, (0.0, 0.0), nanC, nanC)
    assert np.array_equal(r[0], P[0] * 2.0**-5) and np.array_equal(r[1], P[1] * 2.0**-5)
    X_hi = np.array(d["A_hi"][:, :7])
    X_lo = np.zeros_like(X_hi)
    r = orc.i8_casc_gemm_ex("N", "N", (1.0, 0.0), d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"],
                            (1.0, 0.0), X_hi, X_lo)
    for i in range(9):
        for j in range(7):
            ex = fr(P[0][i, j]) + fr(P[1][i, j]) + fr(X_hi[i, j])
            got = fr(r[0][i, j]) + fr(r[1][i, j])
            assert abs(got - ex) <= F(2) ** -104 * (abs(fr(P[0][i, j])) + abs(fr(X_hi[i, j])))
    for alpha, kk in (((1.0, 0.0), 0), ((0.0, 0.0), 300)):
        A = d["A_hi"][:, :kk]
        B = d["B_hi"][:kk]
        r = orc.i8_casc_gemm_ex("N", "N", alpha, A, A, B, B, (2.0, 0.0), X_hi, X_lo)
        assert np.array_equal(r[0], 2 * X_hi) and np.all(r[2] == 0)


@pytest.mark.parametrize("uplo,trans", [("L", "N"), ("U", "T")])
def test_i8_syrk_oracle(orc, uplo, trans):
    """NEXT-4 SYRK on the INT8 cascade: on its triangle within the north-star
    bound of the exact op(A) op(A)^T (exact rationals), the other triangle and
    its flags untouched, alpha = 2^p exact."""
    from fractions import Fraction as F
    n, k = 9, 200
    d = I.make_config(1, m=n, n=k, k=k, seed=21)
    A_hi, A_lo = d["A_hi"][:n, :k], d["A_lo"][:n, :k]
    Ast = (A_hi.T.copy(), A_lo.T.copy()) if trans == "T" else (A_hi.copy(), A_lo.copy())
    sent = np.full((n, n), 3.25)
    fl0 = np.full((n, n), 7, np.uint8)
    Ch, Cl, fl = orc.i8_casc_syrk(uplo, trans, (1.0, 0.0), *Ast, (0.0, 0.0), sent, sent, fl0)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    assert np.all(Ch[~tri] == 3.25) and np.all(fl[~tri] == 7) and np.all(fl[tri] <= 1)
    for i in range(n):
        for j in range(n):
            if not tri[i, j]:
                continue
            a = [F(A_hi[i, p]) + F(A_lo[i, p]) for p in range(k)]
            b = [F(A_hi[j, p]) + F(A_lo[j, p]) for p in range(k)]
            ex = sum(x * z for x, z in zip(a, b))
            absab = sum(abs(x * z) for x, z in zip(a, b))
            assert abs(F(Ch[i, j]) + F(Cl[i, j]) - ex) <= 4 * k * F(2) ** -104 * absab
    S = orc.i8_casc_syrk(uplo, trans, (0.5, 0.0), *Ast, (0.0, 0.0), sent, sent)
    assert np.array_equal(S[0][tri], 0.5 * Ch[tri]) and np.array_equal(S[1][tri], 0.5 * Cl[tri])


@pytest.mark.parametrize("uplo,trans,m,n", [("L", "N", 40, 3), ("U", "T", 300, 2)])
def test_i8_trsm_oracle(orc, uplo, trans, m, n):
    """NEXT-4 TRSM on the INT8 cascade: the exact residual of op(A) X = B within
    2^-90 (|op(A)||X|) row by row for a diagonally dominant A."""
    from fractions import Fraction as F
    rng = np.random.default_rng(31)
    A_hi = rng.uniform(-1, 1, (m, m)) / m
    A_hi = np.tril(A_hi) if uplo == "L" else np.triu(A_hi)
    A_lo = A_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, m))
    dg = 1.0 + rng.uniform(0, 1, m)
    A_hi[np.arange(m), np.arange(m)] = dg
    A_lo[np.arange(m), np.arange(m)] = 0.0
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    X_hi, X_lo = orc.i8_casc_trsm(uplo, "N", (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    A = [[F(A_hi[i, j]) + F(A_lo[i, j]) for j in range(m)] for i in range(m)]
    if trans == "T":
        A = [list(r) for r in zip(*A)]
    lower = (uplo == "L") != (trans == "T")
    for i in range(0, m, 1 if m <= 40 else 11):
        lo, hi = (0, i + 1) if lower else (i, m)
        for j in range(n):
            x = [F(X_hi[l, j]) + F(X_lo[l, j]) for l in range(lo, hi)]
            r = sum(a * b for a, b in zip(A[i][lo:hi], x)) - (F(B_hi[i, j]) + F(B_lo[i, j]))
            mag = sum(abs(a * b) for a, b in zip(A[i][lo:hi], x))
            assert abs(r) <= F(2) ** -90 * mag
