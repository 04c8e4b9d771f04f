"""More pins of the CPU oracle (-m "not gpu"), round 2:

* eq:cascerr and eq:fp642err: `cascerr_bound`
  is pinned to the paper's own specialisation of it, the oracle's error on
  cfg0-2-style data sits under it, the 61-bit guarantee holds wherever bin 0
  is not zero, and the §3.6 worst case breaks that guarantee and is flagged;
* the cross-bin FP64x2 combine (reading R9) bit for bit against its exact
  rational semantics (every TwoSum error term exact, Fast2Sum only where its
  precondition holds, bins in the order 6 -> 0), on hand-built bins where a
  Fast2Sum in place of the first TwoSum, or the order 0 -> 6, gives other
  bits;
* the blocked TRSM (reading R27) against a plain unblocked FP64x2
  substitution that shares none of its block sizes, itself pinned to exact
  rational solutions.
Ground truth is fractions.Fraction and the paper's printed formulas.
"""

import math
import random
from fractions import Fraction as F

import numpy as np
import pytest

import casc_inputs as I

W256 = (22, 21, 21)


def fr(x):
    return F(float(x))


def rn(q):
    """nearest double, ties to even (Python's correctly rounded float(Fraction))"""
    return float(q)


# ----------------------------------------------------------------- eq:cascerr / eq:fp642err
def test_cascerr_bound_matches_papers_specialisation(orc):
    """P:L2899-2916 specialises eq:cascerr to k = 256, D2 + 53 = 117 and bin 0 != 0
    (so |x|^T|y| >= 2^-42 ||x|| ||y||): the bound is <= |x|^T|y| (2^-106 + k 2^-61).
    The oracle's cascerr_bound must reproduce that (it fails with a wrong
    constant 40, a k instead of k^2, or a wrong epsilon)."""
    rng = np.random.default_rng(1)
    nx = rng.uniform(0.5, 1.0, 200)
    ny = rng.uniform(0.5, 1.0, 200)
    absab = nx * ny * 2.0 ** -42 * rng.uniform(1.0, 4.0, 200)  # at the paper's lower limit
    b = orc.cascerr_bound(256, absab, nx, ny, W256)
    assert np.all(b <= absab * (2.0 ** -106 + 256 * 2.0 ** -61))
    # and not loose by more than the paper's rounding of 40 * 2^-67 up to 2^-61
    at_limit = orc.cascerr_bound(256, nx * ny * 2.0 ** -42, nx, ny, W256)
    ratio = at_limit / (nx * ny * 2.0 ** -42 * (2.0 ** -106 + 256 * 2.0 ** -61))
    assert np.all((ratio > 0.6) & (ratio <= 1.0))
    # eps_tilde = 2^-(D2 + 53): 2^-117 at (22, 21, 21)
    one = orc.cascerr_bound(1, 0.0, 1.0, 1.0, W256)
    assert one == 40 * 2.0 ** -117


def _panel_terms(d, p0, p1):
    a, b = np.abs(d["A_hi"][:, p0:p1]), np.abs(d["B_hi"][p0:p1])
    return a @ b * (1 + 2.0 ** -40), a.max(1)[:, None], b.max(0)[None, :]


@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 30, 26, 700), (2, 28, 33, 513),
                                       (3, 16, 12, 1024)])
def test_oracle_error_within_cascerr(orc, cfg, m, n, k):
    """Every entry: |C - C*| <= sum over panels of eq:cascerr (x2 for the terms the
    paper's "approximately" drops) + the FP64x2 rounding of each panel value and
    accumulation step ((2P + 2) 2^-104 |A||B|)."""
    d = I.make_config(cfg, m=m, n=n, k=k, variant="b") if cfg == 3 else \
        I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, _ = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    c = orc.select_widths(k)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo)
    P = -(-k // 256)
    bound = 0.0
    for p0 in range(0, k, 256):
        p1 = min(k, p0 + 256)
        absab, nx, ny = _panel_terms(d, p0, p1)
        bound = bound + 2 * orc.cascerr_bound(p1 - p0, absab, nx, ny, c) \
            + (2 * P + 2) * 2.0 ** -104 * absab
    bound = bound.ravel()
    assert np.all(np.abs(r["err"]) <= bound)
    # the bound is not vacuous: on this data it is within 2^20 of the error seen
    nz = np.abs(r["err"]) > 0
    if nz.any():
        assert np.min(bound[nz] / np.abs(r["err"][nz])) < 2.0 ** 20


@pytest.mark.parametrize("gen", ["uniform", "wide"])
def test_fp642err_where_bin0_nonzero(orc, gen):
    """eq:fp642err: k <= 256 and bin 0 != 0 (flag clear) ->
    |C - C*| <= |x|^T|y| (2^-106 + k 2^-61): at least 61 correct bits."""
    k = 256
    if gen == "uniform":
        d = I.make_config(1, m=40, n=36, k=k, seed=5)
    else:  # rows / columns scaled over 2^+-30 and entries spanning 20 binades
        d = I.make_config(2, m=40, n=36, k=k, seed=6)
        rng = np.random.default_rng(2)
        s = np.ldexp(1.0, rng.integers(-20, 1, (40, k)))
        d["A_hi"], d["A_lo"] = d["A_hi"] * s, d["A_lo"] * s
    C_hi, C_lo, fl = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    ii, jj = np.nonzero(fl == 0)
    assert ii.size > 0
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii, jj, C_hi, C_lo)
    assert np.all(np.abs(r["err"]) <= r["absab"] * (2.0 ** -106 + k * 2.0 ** -61))


def test_worst_case_breaks_61_bits_and_is_flagged(orc):
    """§3.6 worst case x = (1, eps), y = (0, 1): bin 0 vanishes, the
    cascade returns only fl64(eps) -- an error beyond eq:fp642err's 61-bit
    guarantee, which therefore needs bin 0 != 0 -- and the detector flags it."""
    eps_hi = 3e-25  # an FP64x2 eps: 106 bits, of which slice 3 keeps RN(eps)
    eps_lo = math.ldexp(eps_hi, -54) * 0.71875
    A_hi = np.array([[1.0, eps_hi]])
    A_lo = np.array([[0.0, eps_lo]])
    B_hi = np.array([[0.0], [1.0]])
    C_hi, C_lo, fl = orc.casc_gemm(A_hi, A_lo, B_hi, np.zeros((2, 1)))
    eps = fr(eps_hi) + fr(eps_lo)
    err = abs(fr(C_hi[0, 0]) + fr(C_lo[0, 0]) - eps)
    absab = eps  # |x|^T |y|
    assert err > absab * (F(2) ** -106 + 2 * F(2) ** -61)
    assert fl[0, 0] == 1


# ----------------------------------------------------------------- R9 combine, bit for bit
def _two_sum(a, b):
    s = rn(fr(a) + fr(b))
    return s, rn(fr(a) + fr(b) - fr(s))  # the error term is exact (representable)


def _fast_two_sum(a, b):  # Dekker, as the floating-point sequence (valid iff |a| >= |b|)
    s = a + b
    return s, b - (s - a)


def _dd_add_d(h, l, x):
    s, e = _two_sum(h, x)
    e = rn(fr(e) + fr(l))
    return _fast_two_sum(s, e)  # |s| >= |e| here


def r9_model(b0, b1, b2, b36, escale, widths, first="two_sum", order="6to0"):
    """fl_casc with reading R9 in exact rational semantics:
    T = TwoSum(s2 bin2, s3 bin36); T (+)= s1 bin1; T (+)= bin0; T *= 2^escale.
    `first` / `order` build the mutants the pins must reject."""
    D0, D1, D2 = widths[0], widths[0] + widths[1], sum(widths)
    x = [b0, math.ldexp(b1, -D0), math.ldexp(b2, -D1), math.ldexp(b36, -D2)]
    if order == "0to6":
        x = x[::-1]
    pair = _two_sum if first == "two_sum" else _fast_two_sum
    h, l = pair(x[2], x[3])
    h, l = _dd_add_d(h, l, x[1])
    h, l = _dd_add_d(h, l, x[0])
    return math.ldexp(h, escale), math.ldexp(l, escale)


def _hand_built():
    """Bins where the mutants differ from R9 (found by a seeded search over
    integer bins 0-2 and a large bin 3-6, kept verbatim; test below)."""
    return [
        # |s3 bin36| > |s2 bin2| != 0: Fast2Sum(s2 bin2, s3 bin36) loses its error term
        (80.0, 733566.0, -507.0, -2.330459858142828e+22, 0),
        (-270418.0, -22623082379.0, -873.0, -5.637044100322801e+22, 0),
        (-224.0, -9448879903.0, -575697.0, 2.9822777494948886e+22, 0),
        (0.0, 1.0, 1.0000000000000004, -1.3835058055282168e+19, -3),
        # combining bin 0 first (order 0 -> 6) rounds differently
        (-46009623603976.0, 9130610.0, 738119913.0, -2.5482292947405016e+16, 0),
        (-4901247767.0, -8462.0, 4.0, -1956345731594.116, 0),
        (9357439136729.0, 5923932.0, -479498940924.0, 1.0452897947103362e+16, 0),
        # plain cases: bin 0 dominant, all bins comparable, a scale
        (4503599627370497.0, 1048577.0, -2199023255553.0, 9.223372036854774e+18, 1),
        (3.0, 1.0, 1.0, 1.0, 7),
    ]


def test_combine_r9_bitwise(orc):
    """The oracle's combine equals the exact-semantics model of reading R9 bit for
    bit on hand-built and 20000 random bins (bins 0-2 integers below 2^53 as the
    split makes them, bin 3-6 any double, scales across the range)."""
    cases = list(_hand_built())
    rng = random.Random(11)
    for _ in range(20000):
        b0 = float(rng.randint(-2 ** 53 + 1, 2 ** 53 - 1) >> rng.randint(0, 52))
        b1 = float(rng.randint(-2 ** 53 + 1, 2 ** 53 - 1) >> rng.randint(0, 52))
        b2 = float(rng.randint(-2 ** 53 + 1, 2 ** 53 - 1) >> rng.randint(0, 52))
        b36 = rng.choice([-1, 1]) * math.ldexp(rng.random() + 0.5, rng.randint(-10, 70))
        cases.append((b0, b1, b2, b36, rng.randint(-60, 60)))
    for b0, b1, b2, b36, es in cases:
        got = orc.combine(b0, b1, b2, b36, es, W256)
        want = r9_model(b0, b1, b2, b36, es, W256)
        assert np.array_equal(np.array(got).view(np.uint64), np.array(want).view(np.uint64)), \
            (b0, b1, b2, b36, es, got, want)


def test_combine_r9_rejects_mutants():
    """The pins discriminate: on the hand-built bins a Fast2Sum first step, or
    combining bin 0 first (order 0 -> 6), gives other bits than R9 (so the
    bitwise pin above would catch either mistake)."""
    diff_fast = diff_order = 0
    for b in _hand_built():
        ref = r9_model(*b, W256)
        diff_fast += r9_model(*b, W256, first="fast") != ref
        diff_order += r9_model(*b, W256, order="0to6") != ref
    assert diff_fast >= 3 and diff_order >= 3


def test_combine_error_terms_exact(orc):
    """Each T the oracle returns is an exact FP64x2 representation of the
    rounded sum of its inputs: T.hi = RN(T.hi + T.lo) (normalised), and
    |T - exact weighted bin sum| <= 2^-104 |exact| on the hand-built bins where
    Fast2Sum would lose a whole error term."""
    D0, D1, D2 = 22, 43, 64
    for b0, b1, b2, b36, es in _hand_built():
        th, tl = orc.combine(b0, b1, b2, b36, es, W256)
        assert rn(fr(th) + fr(tl)) == th
        ex = (fr(b0) + fr(b1) * F(2) ** -D0 + fr(b2) * F(2) ** -D1 + fr(b36) * F(2) ** -D2) \
            * F(2) ** es
        assert abs(fr(th) + fr(tl) - ex) <= F(2) ** -104 * abs(ex)


# ----------------------------------------------------------------- TRSM vs plain substitution
def _tri_dd(m, uplo, seed, unit=False):
    rng = np.random.default_rng(seed)
    hi = rng.uniform(-1, 1, (m, m)) / m
    hi = np.tril(hi) if uplo == "L" else np.triu(hi)
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, (m, m))
    dg = 1.0 + rng.uniform(0, 1, m)
    hi[np.arange(m), np.arange(m)] = 1.0 if unit else dg
    lo[np.arange(m), np.arange(m)] = 0.0 if unit else dg * 2.0 ** -54
    s = hi + lo
    return s, lo - (s - hi)


@pytest.mark.parametrize("uplo,trans,unit", [("L", "N", False), ("U", "T", True)])
def test_plain_trsm_exact_rationals(orc, uplo, trans, unit):
    """The plain FP64x2 substitution itself: within 2^-100 (|x| + 1) of the exact
    rational solution (12 x 12, three right-hand sides)."""
    m, n = 12, 3
    A_hi, A_lo = _tri_dd(m, uplo, 31, unit)
    rng = np.random.default_rng(4)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    X_hi, X_lo = orc.dd_trsm_plain(uplo, "U" if unit else "N", (1.0, 0.0), A_hi, A_lo, B_hi, B_lo,
                                   trans=trans)
    A = [[fr(A_hi[i, j]) + fr(A_lo[i, j]) for j in range(m)] for i in range(m)]
    if unit:
        for i in range(m):
            A[i][i] = F(1)
    if trans == "T":
        A = [list(r) for r in zip(*A)]
    lower = (uplo == "L") != (trans == "T")
    order = range(m) if lower else range(m - 1, -1, -1)
    for j in range(n):
        x = [F(0)] * m
        for i in order:
            lo, hi = (0, i) if lower else (i + 1, m)
            x[i] = (fr(B_hi[i, j]) + fr(B_lo[i, j]) - sum(A[i][l] * x[l] for l in range(lo, hi))) \
                / A[i][i]
        for i in range(m):
            assert abs(fr(X_hi[i, j]) + fr(X_lo[i, j]) - x[i]) <= F(2) ** -100 * (abs(x[i]) + 1)


@pytest.mark.parametrize("uplo,trans,unit,m,n", [("L", "N", False, 1100, 3), ("U", "N", False, 700, 2),
                                                 ("L", "T", True, 1300, 2), ("U", "T", False, 257, 4)])
def test_blocked_trsm_vs_plain_substitution(orc, uplo, trans, unit, m, n):
    """R27's blocked TRSM (256-row diagonal inverses, 1024-row super-blocks,
    cascaded-GEMM updates) agrees with the plain unblocked substitution to
    2^-92 (|X| + 2^-20) on diagonally dominant systems that span several
    blocks and super-blocks -- a pin that does not depend on the block sizes."""
    A_hi, A_lo = _tri_dd(m, uplo, 13, unit)
    rng = np.random.default_rng(15)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    dg = "U" if unit else "N"
    Xb = orc.casc_trsm(uplo, dg, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    Xp = orc.dd_trsm_plain(uplo, dg, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    diff = np.abs((Xb[0] - Xp[0]) + (Xb[1] - Xp[1]))
    assert np.all(diff <= 2.0 ** -92 * (np.abs(Xp[0]) + 2.0 ** -20))
    # and the comparison is sharp enough to see a 2^-80 error in one row
    bad_lo = Xb[1].copy()
    bad_lo[m // 2] += 2.0 ** -80
    assert np.any(np.abs((Xb[0] - Xp[0]) + (bad_lo - Xp[1])) > 2.0 ** -92 * (np.abs(Xp[0]) + 2.0 ** -20))


# ----------------------------------------------------------------- ORACLE-EXACT, fixed-point form
@pytest.mark.parametrize("cfg,m,n,k", [(1, 40, 30, 300), (2, 50, 40, 513), (1, 64, 64, 1024),
                                       (3, 16, 20, 1024), (0, 64, 64, 64)])
def test_exact_fixed_equals_superaccumulator(orc, cfg, m, n, k):
    """oracle/exact_fixed.py (exact digit GEMMs + integer assembly, used for the
    all-entries cfg1 check) gives the same exact error (C - C*), rounded once,
    as the superaccumulator (orc_exact_entries, itself pinned to Fractions) on
    every entry, for the oracle's own C and for a perturbed C."""
    from oracle import exact_fixed as EF
    d = I.make_config(cfg, m=m, n=n, k=k, variant="b") if cfg == 3 else \
        I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, _ = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    for Cl in (C_lo, C_lo + 2.0 ** -90 * C_hi):
        err, absx = EF.errors(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], C_hi, Cl)
        r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                              C_hi, Cl)
        assert np.array_equal(err.ravel(), r["err"])
        assert np.array_equal(absx.ravel(), np.abs(r["ex_hi"]))  # |RN(C*)|
    with pytest.raises(ValueError):  # one digit GEMM must stay exact
        EF._exact_chunk(np.ones((2, 1025)), np.zeros((2, 1025)), np.ones((1025, 2)),
                        np.zeros((1025, 2)))


@pytest.mark.parametrize("cfg,m,n,k", [(1, 12, 9, 2500), (2, 10, 7, 3000)])
def test_exact_fixed_chunked_k_equals_superaccumulator(orc, cfg, m, n, k):
    """k > 1024: the exact sum of the exact k-chunk products (used for the
    full-size cfg2-4 line checks) equals the superaccumulator's exact error on
    every entry, and all-ones rows give the integer k exactly."""
    from oracle import exact_fixed as EF
    d = I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, _ = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    err, _ = EF.errors(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], C_hi, C_lo)
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo)
    assert np.array_equal(err.ravel(), r["err"])
    one = np.ones((1, k))
    X = EF.exact_product(one, 0 * one, one.T.copy(), 0 * one.T)
    assert X[0, 0] == k << -EF.UNIT_EXP


# ----------------------------------------------------------------- SYMM / TRMM / right TRSM (R28, R29)
def _sym_expand(hi, lo, uplo):
    tri = np.tril(np.ones(hi.shape, bool)) if uplo == "L" else np.triu(np.ones(hi.shape, bool))
    return np.where(tri, hi, hi.T), np.where(tri, lo, lo.T)


@pytest.mark.parametrize("side,uplo,m,n", [("L", "L", 40, 30), ("R", "U", 25, 300), ("L", "U", 260, 5)])
def test_symm_oracle_exact(orc, side, uplo, m, n):
    """SYMM (R28): the other triangle of A is never read (NaN there), and C is
    within the north-star bound of the exact alpha A_sym B (alpha = 1, beta = 0);
    alpha = 2^p, beta = 0 scales exactly; alpha = 0 gives beta C bitwise."""
    ka = m if side == "L" else n
    rng = np.random.default_rng(3)
    d = I.make_config(1, m=ka, n=ka, k=ka, seed=41)
    S_hi, S_lo = _sym_expand(d["A_hi"], d["A_lo"], uplo)
    other = np.triu(np.ones((ka, ka), bool), 1) if uplo == "L" else np.tril(np.ones((ka, ka), bool), -1)
    A_hi = np.where(other, np.nan, d["A_hi"])
    A_lo = np.where(other, np.nan, d["A_lo"])
    B = I.make_config(1, m=m, n=n, k=ka, seed=43)
    B_hi, B_lo = (B["A_hi"], B["A_lo"]) if side == "L" else (B["A_hi"][:, :n], B["A_lo"][:, :n])
    B_hi, B_lo = np.ascontiguousarray(B_hi[:m, :n]), np.ascontiguousarray(B_lo[:m, :n])
    Z = np.zeros((m, n))
    C_hi, C_lo, fl = orc.casc_symm(side, uplo, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, (0.0, 0.0), Z, Z)
    assert np.all(np.isfinite(C_hi))
    L = (S_hi, S_lo, B_hi, B_lo) if side == "L" else (B_hi, B_lo, S_hi, S_lo)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(*L, ii.ravel(), jj.ravel(), C_hi, C_lo)
    assert np.all(np.abs(r["err"]) <= orc.north_star_bound(ka, r["absab"]))
    C2 = orc.casc_symm(side, uplo, (4.0, 0.0), A_hi, A_lo, B_hi, B_lo, (0.0, 0.0), Z, Z)
    assert np.array_equal(C2[0], 4 * C_hi) and np.array_equal(C2[1], 4 * C_lo)
    C0 = rng.uniform(-1, 1, (m, n))
    C3 = orc.casc_symm(side, uplo, (0.0, 0.0), A_hi, A_lo, B_hi, B_lo, (0.5, 0.0), C0, Z)
    assert np.array_equal(C3[0], 0.5 * C0)


@pytest.mark.parametrize("side,uplo,trans,diag,m,n", [("L", "L", "N", "N", 40, 7),
                                                      ("L", "U", "T", "U", 300, 3),
                                                      ("R", "L", "T", "N", 6, 280),
                                                      ("R", "U", "N", "U", 9, 50)])
def test_trmm_oracle_exact(orc, side, uplo, trans, diag, m, n):
    """TRMM (R28): only A's triangle is read (NaN elsewhere, and on the diagonal
    when unit), and B := alpha op(A) B is within the north-star bound of the
    exact product with the triangular matrix."""
    ka = m if side == "L" else n
    d = I.make_config(1, m=ka, n=ka, k=ka, seed=47)
    tri = np.tril(np.ones((ka, ka), bool)) if uplo == "L" else np.triu(np.ones((ka, ka), bool))
    T_hi = np.where(tri, d["A_hi"], 0.0)
    T_lo = np.where(tri, d["A_lo"], 0.0)
    A_hi = np.where(tri, d["A_hi"], np.nan)
    A_lo = np.where(tri, d["A_lo"], np.nan)
    if diag == "U":
        np.fill_diagonal(T_hi, 1.0)
        np.fill_diagonal(T_lo, 0.0)
        np.fill_diagonal(A_hi, np.nan)
        np.fill_diagonal(A_lo, np.nan)
    if trans == "T":
        T_hi, T_lo = T_hi.T.copy(), T_lo.T.copy()
    B = I.make_config(1, m=m, n=n, k=n, seed=49)
    B_hi, B_lo = B["A_hi"], B["A_lo"]
    X_hi, X_lo = orc.casc_trmm(side, uplo, diag, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    assert np.all(np.isfinite(X_hi))
    L = (T_hi, T_lo, B_hi, B_lo) if side == "L" else (B_hi, B_lo, T_hi, T_lo)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(*L, ii.ravel(), jj.ravel(), X_hi, X_lo)
    assert np.all(np.abs(r["err"]) <= orc.north_star_bound(ka, r["absab"]))


@pytest.mark.parametrize("uplo,trans,unit,m,n", [("L", "N", False, 5, 40), ("U", "N", False, 3, 300),
                                                 ("L", "T", True, 4, 600), ("U", "T", False, 2, 1100)])
def test_trsm_right_oracle(orc, uplo, trans, unit, m, n):
    """Right-side TRSM (R29): the exact residual X op(A) - B within 2^-96 |X||op(A)|
    row by row (dyadic rationals), and agreement with the plain unblocked
    substitution on the transposed system to 2^-92."""
    A_hi, A_lo = _tri_dd(n, uplo, 17, unit)
    rng = np.random.default_rng(19)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    dg = "U" if unit else "N"
    X_hi, X_lo = orc.casc_trsm_right(uplo, dg, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    ftr = "N" if trans == "T" else "T"
    P = orc.dd_trsm_plain(uplo, dg, (1.0, 0.0), A_hi, A_lo, B_hi.T.copy(), B_lo.T.copy(), trans=ftr)
    diff = np.abs((X_hi - P[0].T) + (X_lo - P[1].T))
    assert np.all(diff <= 2.0 ** -92 * (np.abs(X_hi) + 2.0 ** -20))
    A = np.array([[fr(A_hi[i, j]) + fr(A_lo[i, j]) for j in range(n)] for i in range(n)], dtype=object) \
        if n <= 300 else None
    if A is not None:
        if unit:
            for i in range(n):
                A[i, i] = F(1)
        opA = A.T if trans == "T" else A
        for i in range(m):
            for j in range(0, n, max(1, n // 25)):
                col = opA[:, j]
                terms = [(fr(X_hi[i, l]) + fr(X_lo[i, l])) * col[l] for l in range(n) if col[l] != 0]
                r = sum(terms) - (fr(B_hi[i, j]) + fr(B_lo[i, j]))
                assert abs(r) <= F(2) ** -96 * sum(abs(t) for t in terms)


@pytest.mark.parametrize("uplo,trans,n,k", [("L", "N", 30, 300), ("U", "T", 25, 513)])
def test_syr2k_oracle_exact(orc, uplo, trans, n, k):
    """SYR2K (R30): the triangle of C within twice the north-star bound of the
    exact op(A) op(B)^T + op(B) op(A)^T (alpha = 1, beta = 0); the other
    triangle untouched; flags = OR of the two products' flags (here: zero rows
    of A flag their row); alpha = 2^p scales exactly."""
    a = I.make_config(1, m=k, n=k, k=k, seed=81)
    b = I.make_config(2, m=k, n=k, k=k, seed=83)
    A_hi, A_lo = a["A_hi"][:n].copy(), a["A_lo"][:n].copy()   # op(A): n x k
    B_hi, B_lo = b["A_hi"][:n].copy(), b["A_lo"][:n].copy()
    A_hi[3] = A_lo[3] = 0.0
    B_hi[3] = B_lo[3] = 0.0
    st = (lambda x: x.T.copy()) if trans == "T" else (lambda x: x)
    C0 = np.full((n, n), 7.0)
    C_hi, C_lo, fl = orc.casc_syr2k(uplo, trans, (1.0, 0.0), st(A_hi), st(A_lo), st(B_hi),
                                    st(B_lo), (0.0, 0.0), C0, np.zeros((n, n)))
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    assert np.all(C_hi[~tri] == 7.0)
    ii, jj = np.nonzero(tri)
    r1 = orc.exact_entries(A_hi, A_lo, B_hi.T.copy(), B_lo.T.copy(), ii, jj)
    r2 = orc.exact_entries(B_hi, B_lo, A_hi.T.copy(), A_lo.T.copy(), ii, jj)
    for t, (i, j) in enumerate(zip(ii, jj)):
        exact = fr(r1["ex_hi"][t]) + fr(r1["ex_lo"][t]) + fr(r2["ex_hi"][t]) + fr(r2["ex_lo"][t])
        bound = 2 * orc.north_star_bound(k, r1["absab"][t] + r2["absab"][t])
        assert abs(fr(C_hi[i, j]) + fr(C_lo[i, j]) - exact) <= F(bound)
    assert np.all(fl[3][tri[3]] == 1) and np.all(fl[:, 3][tri[:, 3]] == 1)
    C2 = orc.casc_syr2k(uplo, trans, (0.25, 0.0), st(A_hi), st(A_lo), st(B_hi), st(B_lo),
                        (0.0, 0.0), C0, np.zeros((n, n)))
    assert np.array_equal(C2[0][tri], 0.25 * C_hi[tri])
