"""The paper's accuracy-study generators (§5.2):
wide-range data and ill-conditioned products.

Input generation only: the double-double helpers below build the
ill-conditioned matrices (a Householder QR and B = Q^T C "in quad arithmetic",
P:L3502-3507, here in FP64x2 — 106 bits instead of FP128's 113, see DESIGN.md
reading R19).  They are not the cascaded method's arithmetic and are used by
neither the CUDA path nor the oracle's method code.

All draws come from the counter-based RNG of casc_inputs (seed, stream, index).
"""

from __future__ import annotations

import numpy as np

from . import _renormalise, uniform01, uniform_pm1

S_WR_EXP = 10      # wide-range: exponent draws
S_WR_SIGN = 11     # wide-range: sign draws
S_WR_VAL = 12      # wide-range: values
S_WR_LO = 13       # wide-range: extra mantissa bits
S_IC_M = 20        # ill-conditioned: random matrix to factor
S_IC_C = 21        # ill-conditioned: small entries of C
S_IC_SIGN = 22     # ill-conditioned: signs
S_IC_ONE = 23      # ill-conditioned: row of the planted 1 per column

_SPLIT = 134217729.0  # 2^27 + 1 (Veltkamp)


# ---------------------------------------------------------------- FP64x2 helpers
def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _split(a):
    t = _SPLIT * a
    hi = t - (t - a)
    return hi, a - hi


def _two_prod(a, b):
    p = a * b
    ah, al = _split(a)
    bh, bl = _split(b)
    return p, ((ah * bh - p) + ah * bl + al * bh) + al * bl


def dd_add(xh, xl, yh, yl):
    s1, s2 = _two_sum(xh, yh)
    t1, t2 = _two_sum(xl, yl)
    s2 = s2 + t1
    s1, s2 = _renormalise(s1, s2)
    s2 = s2 + t2
    return _renormalise(s1, s2)


def dd_mul(xh, xl, yh, yl):
    p, e = _two_prod(xh, yh)
    e = e + (xh * yl + xl * yh)
    return _renormalise(p, e)


def dd_div(xh, xl, yh, yl):
    q1 = xh / yh
    ph, pl = dd_mul(q1, 0.0 * q1, yh, yl)
    rh, rl = dd_add(xh, xl, -ph, -pl)
    q2 = rh / yh
    return _renormalise(q1, q2)


def dd_sqrt(xh, xl):
    s = np.sqrt(xh)
    sh, sl = dd_mul(s, 0.0 * s, s, 0.0 * s)
    rh, rl = dd_add(xh, xl, -sh, -sl)
    return _renormalise(s, rh / (2.0 * s))


def dd_sum(xh, xl, axis=0):
    """Pairwise FP64x2 reduction along `axis`."""
    xh = np.moveaxis(xh, axis, 0)
    xl = np.moveaxis(xl, axis, 0)
    while xh.shape[0] > 1:
        n = xh.shape[0]
        h = n // 2
        sh, sl = dd_add(xh[:h], xl[:h], xh[h:2 * h], xl[h:2 * h])
        if n % 2:
            sh = np.concatenate([sh, xh[2 * h:]])
            sl = np.concatenate([sl, xl[2 * h:]])
        xh, xl = sh, sl
    return xh[0], xl[0]


def dd_matmul(Ah, Al, Bh, Bl, rows_per_chunk: int = 16):
    """FP64x2 GEMM (elementwise two_prod + pairwise reduction over k), in row
    chunks to bound the m x k x n temporaries."""
    m = Ah.shape[0]
    Ch = np.empty((m, Bh.shape[1]))
    Cl = np.empty((m, Bh.shape[1]))
    for r0 in range(0, m, rows_per_chunk):
        r1 = min(m, r0 + rows_per_chunk)
        ph, pl = dd_mul(Ah[r0:r1, :, None], Al[r0:r1, :, None], Bh[None, :, :], Bl[None, :, :])
        Ch[r0:r1], Cl[r0:r1] = dd_sum(ph, pl, axis=1)
    return Ch, Cl


def householder_qr_q(Mh, Ml):
    """Q of the Householder QR of the square FP64x2 matrix M ("FP128 QR
    factorization (using quad Householder transformations)", in FP64x2)."""
    n = Mh.shape[0]
    Rh, Rl = Mh.copy(), Ml.copy()
    Qh, Ql = np.eye(n), np.zeros((n, n))
    for j in range(n - 1):
        xh, xl = Rh[j:, j].copy(), Rl[j:, j].copy()
        sh, sl = dd_mul(xh, xl, xh, xl)
        nh, nl = dd_sqrt(*dd_sum(sh, sl))
        if nh == 0.0:
            continue
        sgn = -1.0 if xh[0] >= 0 else 1.0
        ah, al = sgn * nh, sgn * nl
        vh, vl = xh, xl
        vh[0], vl[0] = dd_add(xh[0], xl[0], -ah, -al)
        th, tl = dd_mul(vh, vl, vh, vl)
        vtv = dd_sum(th, tl)
        bh, bl = dd_div(2.0, 0.0, *vtv)
        # R[j:, j:] -= beta v (v^T R[j:, j:])
        wh, wl = dd_sum(*dd_mul(vh[:, None], vl[:, None], Rh[j:, j:], Rl[j:, j:]), axis=0)
        bvh, bvl = dd_mul(vh, vl, bh, bl)
        uh, ul = dd_mul(bvh[:, None], bvl[:, None], wh[None, :], wl[None, :])
        Rh[j:, j:], Rl[j:, j:] = dd_add(Rh[j:, j:], Rl[j:, j:], -uh, -ul)
        # Q[:, j:] -= (Q[:, j:] v) (beta v)^T   (Q = H_0 H_1 ...)
        zh, zl = dd_sum(*dd_mul(Qh[:, j:], Ql[:, j:], vh[None, :], vl[None, :]), axis=1)
        uh, ul = dd_mul(zh[:, None], zl[:, None], bvh[None, :], bvl[None, :])
        Qh[:, j:], Ql[:, j:] = dd_add(Qh[:, j:], Ql[:, j:], -uh, -ul)
    return Qh, Ql


# ---------------------------------------------------------------- generators
def _idx(nrows, ncols, row0=0):
    r = np.arange(row0, row0 + nrows, dtype=np.uint64)[:, None]
    c = np.arange(ncols, dtype=np.uint64)[None, :]
    return r * np.uint64(ncols) + c


def gen_uniform_dd(seed: int, nrows: int, ncols: int, stream: int = 30):
    """Uniform [-1, 1] FP64 plus random lower mantissa bits."""
    idx = _idx(nrows, ncols)
    h = uniform_pm1(seed, stream, idx)
    l = (h * 2.0 ** -53) * uniform_pm1(seed, stream + 1, idx)
    return _renormalise(h, l)


def gen_widerange(seed: int, m: int, n: int, k: int):
    """Wide-range data: for each row of A and each column of B,
    pick two exponents in [1e-60, 1e20] (decimal, uniform in the exponent) and
    a sign, giving a range [x, y]; fill the row (column) with uniform values in
    it, plus random mantissa bits below 53 (DD).  Reading R20."""
    def ranges(stream_off, count):
        i = np.arange(2 * count, dtype=np.uint64)
        e = -60.0 + 80.0 * uniform01(seed, S_WR_EXP + stream_off, i)
        lo_e, hi_e = np.minimum(e[0::2], e[1::2]), np.maximum(e[0::2], e[1::2])
        sgn = np.where(uniform01(seed, S_WR_SIGN + stream_off, np.arange(count, dtype=np.uint64))
                       < 0.5, -1.0, 1.0)
        return 10.0 ** lo_e, 10.0 ** hi_e, sgn

    def fill(lo, hi, sgn, nrows, ncols, stream_off, by_row):
        idx = _idx(nrows, ncols)
        u = uniform01(seed, S_WR_VAL + stream_off, idx)
        if by_row:
            lo, hi, sgn = lo[:, None], hi[:, None], sgn[:, None]
        else:
            lo, hi, sgn = lo[None, :], hi[None, :], sgn[None, :]
        h = sgn * (lo + (hi - lo) * u)
        l = (h * 2.0 ** -53) * uniform_pm1(seed, S_WR_LO + stream_off, idx)
        return _renormalise(h, l)

    la, ha, sa = ranges(0, m)
    lb, hb, sb = ranges(100, n)
    A_hi, A_lo = fill(la, ha, sa, m, k, 0, True)
    B_hi, B_lo = fill(lb, hb, sb, k, n, 100, False)
    return dict(A_hi=A_hi, A_lo=A_lo, B_hi=B_hi, B_lo=B_lo, m=m, n=n, k=k,
                name=f"widerange_{m}x{n}x{k}")


def gen_illcond(seed: int, n: int, t: float):
    """Ill-conditioned products: A = Q of the QR of a random
    matrix (orthonormal rows), C with entries of magnitude in (t, 10t) and random
    sign plus exactly one 1 per column, B = Q^T C in extended precision, so that
    most entries of A B are cancelling dot products of size ~t."""
    Mh, Ml = gen_uniform_dd(seed, n, n, stream=S_IC_M)
    Qh, Ql = householder_qr_q(Mh, Ml)
    idx = _idx(n, n)
    mag = t * (1.0 + 9.0 * uniform01(seed, S_IC_C, idx))
    sgn = np.where(uniform01(seed, S_IC_SIGN, idx) < 0.5, -1.0, 1.0)
    C = sgn * mag
    one_row = np.floor(uniform01(seed, S_IC_ONE, np.arange(n, dtype=np.uint64)) * n).astype(int)
    C[one_row, np.arange(n)] = 1.0
    Bh, Bl = dd_matmul(Qh.T.copy(), Ql.T.copy(), C, np.zeros_like(C))
    return dict(A_hi=Qh, A_lo=Ql, B_hi=Bh, B_lo=Bl, C_target=C, m=n, n=n, k=n,
                name=f"illcond_t{t:.0e}_{n}")
