"""Seeded fuzz of the fused path against the oracle on random small shapes and
value distributions (ragged tiles and panels, wide exponent ranges, zeros,
full mantissas, in-panel cancellation).  Per case, through the C ABI:
  * slices and scale exponents of every panel bit-exact (casc_split_a / _b vs
    orc.split_{a,b}_panel, +-0 equal);
  * bins 0-2 of every panel bit-exact (casc_debug_bins vs orc.panel_bins);
  * C bitwise the oracle's combine + FP64x2 panel accumulation of the GPU's own
    bins (reading R9 / R10), flags identical to the oracle's (both modes:
    split mode where the plan picks it, and per tile).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

KINDS = ("uniform", "wide", "sparse", "fullmant", "cancel")


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


def same_values(x, y):  # +-0 equal
    return bool(np.all(x == y))


def _pairs(rng, shape, kind):
    """FP64x2 pairs (hi, lo), |lo| <= ulp(hi)/2 (renormalised by Fast2Sum)."""
    hi = rng.uniform(-1.0, 1.0, shape)
    if kind == "fullmant":  # (1 + u) 2^-L, L up to 40 binades below 1
        hi = np.ldexp(rng.uniform(1.0, 2.0, shape), -rng.integers(1, 41, shape)) * \
            rng.choice([-1.0, 1.0], shape)
    if kind == "sparse":
        hi[rng.random(shape) < 0.4] = 0.0
    lo = hi * 2.0**-53 * rng.uniform(-1.0, 1.0, shape)
    s = hi + lo
    return s, lo - (s - hi)


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    kind = KINDS[seed % len(KINDS)]
    m, n = int(rng.integers(1, 97)), int(rng.integers(1, 97))
    k = int(rng.integers(1, 801))
    A_hi, A_lo = _pairs(rng, (m, k), kind)
    B_hi, B_lo = _pairs(rng, (k, n), kind)
    if kind == "wide":  # rows of A / columns of B scaled by 2^[-100, 100]
        u = rng.integers(-100, 101, m)[:, None]
        v = rng.integers(-100, 101, n)[None, :]
        A_hi, A_lo, B_hi, B_lo = (np.ldexp(A_hi, u), np.ldexp(A_lo, u), np.ldexp(B_hi, v),
                                  np.ldexp(B_lo, v))
    if kind == "cancel" and k >= 2:  # in-panel pairing: B[p+h] = -B[p] for the first h of a panel
        for p0 in range(0, k, 256):
            w = min(256, k - p0)
            h = w // 2
            A_hi[:, p0 + h:p0 + 2 * h] = A_hi[:, p0:p0 + h]
            A_lo[:, p0 + h:p0 + 2 * h] = A_lo[:, p0:p0 + h]
            B_hi[p0 + h:p0 + 2 * h] = -B_hi[p0:p0 + h]
            B_lo[p0 + h:p0 + 2 * h] = -B_lo[p0:p0 + h]
    return kind, m, n, k, A_hi, A_lo, B_hi, B_lo


@pytest.mark.parametrize("seed", range(20))
def test_fuzz_against_oracle(casc, orc, seed):
    kind, m, n, k, A_hi, A_lo, B_hi, B_lo = _case(seed)
    c = orc.select_widths(k)
    args = [T(A_hi), T(A_lo), T(B_hi), T(B_lo)]
    ref_hi = np.zeros((m, n))
    ref_lo = np.zeros((m, n))
    ref_fl = np.zeros((m, n), dtype=np.uint8)
    SA, ge = (N(x) for x in casc.casc_split_a(args[0], args[1]))
    SB, gf = (N(x) for x in casc.casc_split_b(args[2], args[3]))
    assert casc.casc_select_widths(k) == c
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        oa, e = orc.split_a_panel(A_hi[:, p0:p1], A_lo[:, p0:p1], c)
        ob, f = orc.split_b_panel(B_hi[p0:p1], B_lo[p0:p1], c)
        assert np.array_equal(ge[q], e) and np.array_equal(gf[q], f), kind
        assert same_values(SA[:, :, p0:p1], oa) and same_values(SB[:, p0:p1, :], ob), kind
        gb = N(casc.casc_debug_bins(*args, q))
        ob_bins = orc.panel_bins(oa, ob, c)
        for b in range(3):
            assert same_values(gb[b], ob_bins[b]), f"{kind} bin {b} panel {q}"
        for i in range(m):
            for j in range(n):
                th, tl = orc.combine(gb[0, i, j], gb[1, i, j], gb[2, i, j], gb[3, i, j],
                                     int(e[i]) + int(f[j]), c)
                ref_hi[i, j], ref_lo[i, j] = orc.dd_add(ref_hi[i, j], ref_lo[i, j], th, tl)
                ref_fl[i, j] |= gb[0, i, j] == 0.0
    o_fl = orc.casc_gemm(A_hi, A_lo, B_hi, B_lo)[2]
    assert np.array_equal(ref_fl, o_fl), kind
    bits = lambda x: np.ascontiguousarray(x).view(np.uint64)
    for mode in ("1", "0"):
        os.environ["CASC_SPLIT_MODE"] = mode
        try:
            C_hi, C_lo, fl = (N(x) for x in casc.casc_gemm_fp64x2(*args))
        finally:
            del os.environ["CASC_SPLIT_MODE"]
        assert np.array_equal(bits(C_hi), bits(ref_hi)), (kind, mode)
        assert np.array_equal(bits(C_lo), bits(ref_lo)), (kind, mode)
        assert np.array_equal(fl, o_fl), (kind, mode)


@pytest.mark.parametrize("seed", range(12))
def test_i8_fuzz_against_oracle(casc, orc, seed):
    """The INT8 cascade (NEXT-3) on the same kinds of inputs, random slice
    counts y and one k beyond the 8192 panel: C, flags bitwise its oracle's."""
    kind, m, n, k, A_hi, A_lo, B_hi, B_lo = _case(seed)
    rng = np.random.default_rng(2000 + seed)
    y = int(rng.integers(3, 16))
    if seed % 4 == 3:  # two panels of the INT8 cascade (R22)
        kind2, m, n, _, A_hi, A_lo, B_hi, B_lo = _case(100 + seed)
        k = 8192 + int(rng.integers(1, 300))
        m, n = min(m, 24), min(n, 24)
        A_hi, A_lo = _pairs(rng, (m, k), kind2)
        B_hi, B_lo = _pairs(rng, (k, n), kind2)
    args = [T(A_hi), T(A_lo), T(B_hi), T(B_lo)]
    C_hi, C_lo, fl = (N(x) for x in casc.casc_i8_gemm_fp64x2(*args, y=y))
    o_hi, o_lo, o_fl = orc.i8_casc_gemm(A_hi, A_lo, B_hi, B_lo, y)
    bits = lambda x: np.ascontiguousarray(x).view(np.uint64)
    assert np.array_equal(bits(C_hi), bits(o_hi)), (kind, y, m, n, k)
    assert np.array_equal(bits(C_lo), bits(o_lo)), (kind, y, m, n, k)
    assert np.array_equal(fl, o_fl), (kind, y)
