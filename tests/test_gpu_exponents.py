"""GPU parity over the whole binary64 exponent range (reading R16).

FP64x2 has no more exponent range than FP64 (§3.1), and the
method applies its per-row / per-column scales 2^-e (split, App. A
P:L3952-3985) and 2^(e_i+f_j) (combine) by power-of-two
multiplication; the oracle does both with C99 ldexp (one rounding, subnormal
grid, overflow to +-inf).  The kernels must agree bit for bit wherever a
power 2^n falls outside the normal doubles:

* the device scaling itself, against numpy's ldexp on every kind of x / n;
* split slices and exponents (rows scaled so that -e leaves [-1022, 1023]);
* the fused kernel's combine (e_i + f_j near -1030, -15, +1020, +1040 and
  beyond: subnormal and overflowing C), in both the one-item-per-tile mode and
  the small-problem split mode;
* the simple path's standalone epilogue, on bins rebuilt from its own slice
  products.
Each is compared bitwise with the oracle's combine of the GPU's own bins (bin 3-6
is order-dependent, reading R17), flags with the oracle's, and C with the exact
product where it is representable.
"""

import os

import numpy as np
import pytest

import casc_inputs as I

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def casc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2303_04353_b200 as casc
    return casc


def T(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def N(t):
    return t.cpu().numpy()


def bits(x):
    return np.ascontiguousarray(x).view(np.uint64)


# ------------------------------------------------------------------ the scaling itself
def test_ldexp_bitwise(casc):
    rng = np.random.default_rng(5)
    cnt = 200000
    mant = rng.uniform(1.0, 2.0, cnt) * rng.choice([-1.0, 1.0], cnt)
    ex = rng.integers(-1074, 1024, cnt)
    x = np.ldexp(mant, ex)
    # every class of x: zeros of both signs, min / max subnormal, min normal,
    # max finite, ties on the subnormal grid
    special = np.array([0.0, -0.0, 5e-324, -5e-324, 2.0 ** -1022 - 2.0 ** -1074, 2.0 ** -1022,
                        np.finfo(np.float64).max, -np.finfo(np.float64).max, 1.0, 1.5, -1.5,
                        3.0 * 2.0 ** -1000, 1.0 + 2.0 ** -52, 2.0 ** 1023, 0.75])
    x[:special.size] = special
    n = rng.integers(-2300, 2300, cnt)
    # exponents around every boundary of the fast path and of the slow path's cases
    edges = np.array([-2200, -2150, -2098, -2097, -2096, -2095, -2046, -2045, -1100, -1075, -1074,
                      -1073, -1024, -1023, -1022, -1021, 0, 1022, 1023, 1024, 1025, 2046, 2047,
                      2048, 3000])
    n[:special.size * edges.size] = np.tile(edges, special.size)
    x[:special.size * edges.size] = np.repeat(special, edges.size)
    # results landing exactly on subnormal rounding ties: x = (2j + 1) 2^-1075 * 2^s
    j = rng.integers(0, 2 ** 20, 2000)
    s = rng.integers(1, 1000, 2000)
    x[-2000:] = np.ldexp((2 * j + 1).astype(np.float64), -1075 + s)
    n[-2000:] = -s
    got = N(casc.casc_debug_ldexp(T(x), T(n.astype(np.int32))))
    want = np.ldexp(x, n)
    bad = np.nonzero(bits(got) != bits(want))[0]
    assert bad.size == 0, [(x[i], int(n[i]), got[i], want[i]) for i in bad[:5]]


# ------------------------------------------------------------------ inputs
ROW_SHIFT = [-1060, -515, 0, 500, 520, 1000]     # 2^u per row of A
COL_SHIFT = [-515, 0, 520, -1000, 23]            # 2^v per column of B


def _scaled(m, n, k, seed, big_rows=()):
    """cfg1-style data with rows of A scaled by 2^u_i and columns of B by 2^v_j
    (cycling through ROW_SHIFT / COL_SHIFT), renormalised pairs; the rows in
    big_rows get one element of magnitude 1.5 2^1023 (panel max >= 2^1023)."""
    d = I.make_config(1, m=m, n=n, k=k, seed=seed)
    u = np.array([ROW_SHIFT[i % len(ROW_SHIFT)] for i in range(m)])
    v = np.array([COL_SHIFT[j % len(COL_SHIFT)] for j in range(n)])
    A_hi, A_lo = np.ldexp(d["A_hi"], u[:, None]), np.ldexp(d["A_lo"], u[:, None])
    B_hi, B_lo = np.ldexp(d["B_hi"], v[None, :]), np.ldexp(d["B_lo"], v[None, :])
    for r in big_rows:
        A_hi[r, 3] = 1.5 * 2.0 ** 1023
        A_lo[r, 3] = 0.0
    # renormalise (scaling by 2^u keeps pairs normalised except where lo underflowed)
    s = A_hi + A_lo
    A_lo, A_hi = A_lo - (s - A_hi), s
    s = B_hi + B_lo
    B_lo, B_hi = B_lo - (s - B_hi), s
    return dict(A_hi=A_hi, A_lo=A_lo, B_hi=B_hi, B_lo=B_lo, m=m, n=n, k=k)


def _same(x, y):
    return bool(np.all((x == y) | (np.isnan(x) & np.isnan(y))))


def _oracle_combined(orc, d, bins_of_panel):
    """C and flags from the oracle's combine (ldexp scaling) + FP64x2 panel
    accumulation applied to given bins (4 x m x n per panel, paper scales)."""
    m, n, k = d["m"], d["n"], d["k"]
    c = orc.select_widths(k)
    ref_hi = np.zeros((m, n))
    ref_lo = np.zeros((m, n))
    ref_fl = np.zeros((m, n), dtype=np.uint8)
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        gb = bins_of_panel(q)
        _, e = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        _, f = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        for i in range(m):
            for j in range(n):
                th, tl = orc.combine(gb[0, i, j], gb[1, i, j], gb[2, i, j], gb[3, i, j],
                                     int(e[i]) + int(f[j]), c)
                if q == 0:
                    ref_hi[i, j], ref_lo[i, j] = orc.dd_add(0.0, 0.0, th, tl)
                else:
                    ref_hi[i, j], ref_lo[i, j] = orc.dd_add(ref_hi[i, j], ref_lo[i, j], th, tl)
                ref_fl[i, j] |= gb[0, i, j] == 0.0
    return ref_hi, ref_lo, ref_fl


def _escales(orc, d):
    c = orc.select_widths(d["k"])
    _, e = orc.split_a_panel(d["A_hi"][:, :256], d["A_lo"][:, :256], c)
    _, f = orc.split_b_panel(d["B_hi"][:256], d["B_lo"][:256], c)
    return e[:, None].astype(int) + f[None, :].astype(int)


# ------------------------------------------------------------------ split
def test_split_extreme_exponents_bit_exact(casc, orc):
    d = _scaled(30, 25, 300, seed=41, big_rows=(5, 11))
    SA, e = casc.casc_split_a(T(d["A_hi"]), T(d["A_lo"]))
    SB, f = casc.casc_split_b(T(d["B_hi"]), T(d["B_lo"]))
    SA, e, SB, f = N(SA), N(e), N(SB), N(f)
    c = orc.select_widths(300)
    for q, p0 in enumerate(range(0, 300, 256)):
        p1 = min(300, p0 + 256)
        oa, oe = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        ob, of = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        assert np.array_equal(e[q], oe) and np.array_equal(f[q], of)
        assert _same(SA[:, :, p0:p1], oa) and _same(SB[:, p0:p1, :], ob)
    # the wide scalings were exercised: -e outside [-1022, 1023]
    assert (e < -1023).any() and (e == 1024).any()


# ------------------------------------------------------------------ fused combine
def test_fused_combine_extreme_exponents_bitwise(casc, orc):
    """C of the fused kernel == the oracle's combine (ldexp per limb) of the
    GPU's own bins, bit for bit, with e_i + f_j across the whole range."""
    d = _scaled(24, 20, 300, seed=43, big_rows=(11,))
    es = _escales(orc, d)
    assert (es < -1022).any() and (es > 1023).any() and ((es >= -1022) & (es <= 1023)).any()
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    C_hi, C_lo, flags = (N(x) for x in casc.casc_gemm_fp64x2(*args))
    ref_hi, ref_lo, ref_fl = _oracle_combined(
        orc, d, lambda q: N(casc.casc_debug_bins(*args, q)))
    assert _same(C_hi, ref_hi) and _same(C_lo, ref_lo)
    assert np.array_equal(bits(C_hi), bits(ref_hi)) and np.array_equal(bits(C_lo), bits(ref_lo))
    assert np.array_equal(flags, ref_fl)
    # subnormal and overflowing results occur (an overflowing panel value is
    # +-inf, and the FP64x2 additions after it turn it into NaN on both sides)
    assert (np.abs(C_hi[np.isfinite(C_hi)]) < 2.0 ** -1022).any() and (~np.isfinite(C_hi)).any()
    _check_vs_exact_and_oracle(orc, d, C_hi, C_lo, flags)


def _cascerr_total(orc, d):
    """Sum over the k panels of eq:cascerr for every entry:
    |x|^T|y| 2^-106 + 40 k^2 2^-(D2+53) ||x||_inf ||y||_inf per panel row /
    column segment, doubled for the terms the paper's "approximately" drops,
    plus the FP64x2 rounding of each panel value and accumulation step
    ((2P + 2) 2^-104 |A||B|).  With rows of huge dynamic range (a 2^1023
    element beside 2^520 ones) only this bound applies: the small elements
    are carried by slice 3 with FP64 accuracy (reading R6)."""
    k = d["k"]
    c = orc.select_widths(k)
    tot = 0.0
    P = -(-k // 256)
    with np.errstate(over="ignore", under="ignore", invalid="ignore"):
        for p0 in range(0, k, 256):
            p1 = min(k, p0 + 256)
            a, b = np.abs(d["A_hi"][:, p0:p1]), np.abs(d["B_hi"][p0:p1])
            absab = (a @ b) * (1 + 2.0 ** -40)
            tot = tot + 2 * orc.cascerr_bound(p1 - p0, absab, a.max(1)[:, None],
                                              b.max(0)[None, :], c) \
                + (2 * P + 2) * 2.0 ** -104 * absab
    return tot.ravel()


def _check_vs_exact_and_oracle(orc, d, C_hi, C_lo, flags):
    """Flags equal the oracle's; wherever the exact product and C are finite
    normal-range values, C is within the north-star bound or eq:cascerr (their
    sum bounds both) plus the absolute error of the subnormal grid."""
    m, n, k = d["m"], d["n"], d["k"]
    o_hi, o_lo, o_fl = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    assert np.array_equal(flags, o_fl)
    P = -(-k // 256)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo)
    fin = np.isfinite(C_hi.ravel()) & (np.abs(r["ex_hi"]) < 2.0 ** 1023)
    # gradual underflow: an FP64x2 value near 2^-1000 keeps only ~74 bits (its lo
    # limb is subnormal), and every rounding of such a limb in the combine, the
    # scaling and the accumulation loses up to an ulp of 2^-1074; the oracle
    # itself shows up to ~11 of them per panel on these inputs
    bound = orc.north_star_bound(k, r["absab"]) + _cascerr_total(orc, d) \
        + 16 * (P + 1) * 2.0 ** -1074
    assert np.all(np.abs(r["err"][fin]) <= bound[fin])
    # overflow: C is non-finite exactly where the oracle's is
    assert np.array_equal(np.isfinite(C_hi), np.isfinite(o_hi))
    both = np.isfinite(o_hi).ravel()
    diff = np.abs((C_hi.ravel() - o_hi.ravel()) + (C_lo.ravel() - o_lo.ravel()))
    assert np.all(diff[both & fin] <= 2 * bound[both & fin])


def test_split_mode_extreme_exponents_bitwise(casc):
    """Small-problem split mode (one work item per (tile, panel) + ordered
    reduction) on the same ranges: bitwise the one-item-per-tile result."""
    d = _scaled(256, 256, 1024, seed=47, big_rows=(7, 130))
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    split = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    os.environ["CASC_SPLIT_MODE"] = "0"
    try:
        whole = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    finally:
        del os.environ["CASC_SPLIT_MODE"]
    for a, b in zip(split, whole):
        assert np.array_equal(bits(a) if a.dtype == np.float64 else a,
                              bits(b) if b.dtype == np.float64 else b)


@pytest.mark.parametrize("m,n,k", [(24, 20, 300), (256, 256, 1024)])
def test_blas_ex_extreme_exponents(casc, orc, m, n, k):
    """The BLAS-style instantiation (alpha / beta applied at the last panel, or
    in the split-mode reduction for the second shape) scales the same way:
    alpha = 1, beta = 0 give bitwise the plain product; a beta update reads the
    ORIGINAL C also for the elements the WIDE re-run computes, and equals the
    oracle's FP64x2 update of the plain product bit for bit."""
    import torch
    d = _scaled(m, n, k, seed=53, big_rows=(5,))
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    ref = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    C_hi = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    C_lo = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    casc.casc_gemm_fp64x2_ex("T", "N", 1.0, T(d["A_hi"].T.copy()), T(d["A_lo"].T.copy()),
                             args[2], args[3], 0.0, C_hi, C_lo)
    assert np.array_equal(bits(N(C_hi)), bits(ref[0])) and np.array_equal(bits(N(C_lo)), bits(ref[1]))
    rng = np.random.default_rng(3)
    C0 = np.ldexp(rng.uniform(-1, 1, (m, n)), rng.integers(-1000, 1000, (m, n)))
    al, be = (0.75, 2.0 ** -60), (-1.5, 0.0)
    C_hi, C_lo = T(C0), T(np.zeros((m, n)))
    casc.casc_gemm_fp64x2_ex("N", "N", al, *args, be, C_hi, C_lo)
    g_hi, g_lo = N(C_hi), N(C_lo)
    for i in range(0, m, max(1, m // 24)):
        for j in range(0, n, max(1, n // 20)):
            th, tl = orc.dd_mul(al[0], al[1], ref[0][i, j], ref[1][i, j])
            uh, ul = orc.dd_mul(be[0], be[1], C0[i, j], 0.0)
            th, tl = orc.dd_add(th, tl, uh, ul)
            assert bits(np.array([g_hi[i, j], g_lo[i, j]])).tolist() == \
                bits(np.array([th, tl])).tolist(), (i, j)


def test_syrk_extreme_exponents(casc):
    """SYRK's triangular instantiation: every stored element bitwise the GEMM's."""
    import torch
    d = _scaled(130, 300, 300, seed=61, big_rows=(2,))
    A_hi, A_lo = d["A_hi"], d["A_lo"]
    G_hi = torch.zeros((130, 130), dtype=torch.float64, device="cuda")
    G_lo = torch.zeros((130, 130), dtype=torch.float64, device="cuda")
    casc.casc_gemm_fp64x2_ex("N", "T", 1.0, T(A_hi), T(A_lo), T(A_hi), T(A_lo), 0.0, G_hi, G_lo)
    S_hi = torch.full((130, 130), float("nan"), dtype=torch.float64, device="cuda")
    S_lo = torch.full((130, 130), float("nan"), dtype=torch.float64, device="cuda")
    casc.casc_syrk_fp64x2("L", "N", 1.0, T(A_hi), T(A_lo), 0.0, S_hi, S_lo)
    tri = np.tril(np.ones((130, 130), bool))
    assert np.array_equal(bits(N(S_hi)[tri]), bits(N(G_hi)[tri]))
    assert np.array_equal(bits(N(S_lo)[tri]), bits(N(G_lo)[tri]))
    assert np.all(np.isnan(N(S_hi)[~tri]))


# ------------------------------------------------------------------ simple path
PRODUCTS = [(0, 0, 0), (1, 0, 1), (1, 1, 0), (2, 0, 2), (2, 1, 1), (2, 2, 0), (3, 0, 3), (3, 1, 4),
            (3, 2, 5), (3, 3, 6)]


def test_simple_path_extreme_exponents_bitwise(casc, orc):
    """§4.2 simple path: its standalone epilogue equals the oracle's combine of
    its own bins.  The bins are rebuilt from the path's slice GEMMs
    (casc_slice_product, paper normalisation): bins 0-2 are exact sums; bin 3-6
    is accumulated in the simple path's order ((P03 + s P14) + s P25) + P36,
    s = 2^(c2 - c0) (the pre-alignment, exact)."""
    d = _scaled(20, 18, 300, seed=59, big_rows=(3,))
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    c = orc.select_widths(300)
    s = 2.0 ** (c[2] - c[0])
    s1 = 2.0 ** (c[1] - c[0])  # bin 2 = A0 B2 + 2^(c1-c0) A1 B1 + A2 B0 (reading R8)

    def bins_of_panel(q):
        P = {(sa, sb): N(casc.casc_slice_product(*args, sa, sb, q)) for _, sa, sb in PRODUCTS}
        b0 = P[0, 0]
        b1 = P[0, 1] + P[1, 0]                                     # exact
        b2 = P[0, 2] + s1 * P[1, 1] + P[2, 0]                      # exact
        b36 = ((P[0, 3] + s * P[1, 4]) + s * P[2, 5]) + P[3, 6]    # the path's order
        return np.stack([b0, b1, b2, b36])

    C_hi, C_lo, flags = (N(x) for x in casc.casc_gemm_fp64x2_simple(*args))
    ref_hi, ref_lo, ref_fl = _oracle_combined(orc, d, bins_of_panel)
    assert np.array_equal(bits(C_hi), bits(ref_hi)) and np.array_equal(bits(C_lo), bits(ref_lo))
    assert np.array_equal(flags, ref_fl)
    _check_vs_exact_and_oracle(orc, d, C_hi, C_lo, flags)


@pytest.mark.parametrize("m,n,k", [(256, 256, 512), (640, 576, 300)])
def test_all_elements_wide_bitwise(casc, orc, m, n, k):
    """Every scale outside the normal powers of two (A, B ~ 2^-520: subnormal
    C): every warp of every item is re-run once by the WIDE launch (one list
    entry per item, a warp mask), in split mode (first shape) and per tile
    (second); C bitwise the oracle's combine of the GPU's own bins."""
    d = I.make_config(1, m=m, n=n, k=k, seed=67)
    for x in ("A_hi", "A_lo", "B_hi", "B_lo"):
        d[x] = np.ldexp(d[x], -520)
    d["m"], d["n"], d["k"] = m, n, k
    assert (_escales(orc, d) < -1022).all()
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    C_hi, C_lo, flags = (N(x) for x in casc.casc_gemm_fp64x2(*args))
    ref_hi, ref_lo, ref_fl = _oracle_combined(orc, d, lambda q: N(casc.casc_debug_bins(*args, q)))
    assert np.array_equal(bits(C_hi), bits(ref_hi)) and np.array_equal(bits(C_lo), bits(ref_lo))
    assert np.array_equal(flags, ref_fl)
    assert (C_hi != 0).any()


def test_all_wide_costs_one_rerun(casc):
    """The all-wide case recomputes each item once (not once per warp): at
    2048^3 it takes less than 2.5x the time of the same call on normal scales."""
    import torch
    n = 2048
    d = I.make_config(1, m=n, n=n, k=n, seed=69)
    norm = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    wide = [T(np.ldexp(d[x], -520)) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    C = [torch.empty((n, n), dtype=torch.float64, device="cuda") for _ in range(2)]
    ws = torch.empty(casc.casc_workspace_bytes(n, n, n), dtype=torch.uint8, device="cuda")

    def t(args):
        casc.casc_gemm_fp64x2(*args, C_hi=C[0], C_lo=C[1], workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            casc.casc_gemm_fp64x2(*args, C_hi=C[0], C_lo=C[1], workspace=ws)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / 3
    t_norm, t_wide = t(norm), t(wide)
    assert t_wide < 2.5 * t_norm, (t_norm, t_wide)


def test_split_mode_mixed_wide_panels_bitwise(casc, orc):
    """Split mode with the fold inside the product launch: a (tile, warp) whose
    scales leave the normal powers of two in ONE panel only (rows of A and
    rows of B in panel 1 scaled by 2^-600 / 2^-500: e + f < -1022 there) is
    folded by the WIDE re-run, the others by the product launch.  C and the
    flags are bitwise the per-tile mode's and the oracle's combine of the
    GPU's own bins; an alpha / beta update likewise."""
    import torch
    m, n, k = 128, 192, 768
    d = I.make_config(1, m=m, n=n, k=k, seed=71)
    rows = np.arange(m) % 3 == 0
    for x in ("A_hi", "A_lo"):
        d[x][rows, 256:512] = np.ldexp(d[x][rows, 256:512], -600)
    for x in ("B_hi", "B_lo"):
        d[x][256:512, :] = np.ldexp(d[x][256:512, :], -500)
    d["m"], d["n"], d["k"] = m, n, k
    c = orc.select_widths(k)
    _, e1 = orc.split_a_panel(d["A_hi"][:, 256:512], d["A_lo"][:, 256:512], c)
    _, f1 = orc.split_b_panel(d["B_hi"][256:512], d["B_lo"][256:512], c)
    es1 = e1[:, None].astype(int) + f1[None, :].astype(int)
    assert (es1 < -1022).any() and (es1 >= -1022).any() and (_escales(orc, d) >= -1022).all()
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    split = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    os.environ["CASC_SPLIT_MODE"] = "0"
    try:
        whole = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    finally:
        del os.environ["CASC_SPLIT_MODE"]
    for a, b in zip(split, whole):
        assert np.array_equal(bits(a) if a.dtype == np.float64 else a,
                              bits(b) if b.dtype == np.float64 else b)
    ref_hi, ref_lo, ref_fl = _oracle_combined(orc, d, lambda q: N(casc.casc_debug_bins(*args, q)))
    assert np.array_equal(bits(split[0]), bits(ref_hi)) and np.array_equal(bits(split[1]),
                                                                            bits(ref_lo))
    assert np.array_equal(split[2], ref_fl)
    al, be = (0.75, 2.0**-60), (1.5, 0.0)
    C0 = np.random.default_rng(5).uniform(-1, 1, (m, n))
    outs = []
    for mode in ("1", "0"):
        os.environ["CASC_SPLIT_MODE"] = mode
        try:
            C_hi, C_lo = T(C0), T(np.zeros((m, n)))
            fl = torch.full((m, n), 7, dtype=torch.uint8, device="cuda")
            casc.casc_gemm_fp64x2_ex("N", "N", al, *args, be, C_hi, C_lo, flags=fl)
            outs.append((bits(N(C_hi)), bits(N(C_lo)), N(fl)))
        finally:
            del os.environ["CASC_SPLIT_MODE"]
    for a, b in zip(*outs):
        assert np.array_equal(a, b)
