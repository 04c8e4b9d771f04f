"""ORACLE-EXACT in fixed-point slice form: the exact product C* = A B of FP64x2
matrices for EVERY entry of a full-size problem (TEST INFRASTRUCTURE ONLY,
like the rest of oracle/).

The superaccumulator of casc_oracle.c (orc_exact_entries) costs ~1 ms per
entry at k = 1024, too slow for all 10^6 entries of BASELINE cfg1 (SURVEY
§8(d): "all 1M entries checked exactly").  This evaluator gets the same exact
values from exact integer arithmetic instead:

1. Each row of A (column of B) is scaled by the power of two 2^-s of its
   largest |hi| (exact), so its entries lie in (-1, 1).
2. Each limb is cut into signed base-2^20 digits by repeated exact
   trunc(x 2^20) (every step is an exact binary64 operation); the hi and lo
   digits are added, so a value is x = sum_s d_s 2^(-20 (s+1)) with integer
   |d_s| < 2^21, and the cut is checked to leave no remainder.
3. For every digit pair (s, t) the integer matrix product D^A_s D^B_t is a
   library GEMM (numpy float64): all its partial sums are integers below
   2^21 * 2^21 * k <= 2^52 for k <= 1024, so it is EXACT in any summation
   order (the step the plan allows: "a library primitive (a matmul) may serve
   as a step").
4. The products of each anti-diagonal d = s + t are added in int64, and the
   exact value of every entry is assembled as a Python integer in units of
   2^-1100 (every binary64 number is an integer multiple of 2^-1074), with
   the row / column scales applied as shifts.
5. k > 1024: C* = sum over k-chunks of 1024 of the chunks' exact products,
   each assembled as above (its own row / column scales) in the same integer
   units, added as Python integers -- exact, so the chunking is invisible.
Pinned against the superaccumulator (tests/test_oracle_bounds.py): equal
RN(C*) (hi, lo) bit for bit on sampled entries of cfg1 / cfg2-style data,
also with k > 1024.
"""

from __future__ import annotations

import numpy as np

DIGIT = 20         # bits per digit
UNIT_EXP = -1100   # exact integer unit of the assembled values
MAX_K = 1024       # 2^21 * 2^21 * k < 2^53 keeps every digit GEMM exact


def _row_scale(hi):
    """power-of-two exponent s per row with max |hi| < 2^s (0 for zero rows)"""
    mx = np.abs(hi).max(axis=1)
    _, e = np.frexp(mx)
    return np.where(mx > 0, e, 0).astype(np.int64)


def _digits(x, nd):
    """signed base-2^20 digits of x (rows scaled into (-1, 1)): nd arrays with
    x = sum_s d_s 2^(-20 (s+1)); raises if x needs more digits."""
    a = x.copy()
    out = []
    for _ in range(nd):
        a = a * 2.0 ** DIGIT          # exact (power of two, no overflow: |a| < 2^20)
        d = np.trunc(a)               # exact; toward zero, so that
        a = a - d                     # the fraction keeps a's sign and is exact
        out.append(d)
    if np.any(a != 0):
        raise ValueError("exact_fixed: entries need more digits than allowed")
    return out


def _needed_digits(*limbs):
    """digits needed to hold every (scaled, |x| < 1) limb exactly: its lowest
    set bit is >= 2^(e - 53) for x = m 2^e, m in [0.5, 1)"""
    lowest = 0
    for x in limbs:
        nz = x != 0
        if nz.any():
            _, e = np.frexp(x[nz])
            lowest = min(lowest, int(e.min()) - 53)
    return max(1, -(lowest // DIGIT))


def exact_product(A_hi, A_lo, B_hi, B_lo):
    """Exact C* = (A_hi + A_lo)(B_hi + B_lo) for every entry, as an object array
    of Python ints in units of 2^UNIT_EXP (m x n); k > 1024 in exact chunks."""
    k = A_hi.shape[1]
    X = None
    for p0 in range(0, max(k, 1), MAX_K):
        p1 = min(k, p0 + MAX_K)
        part = _exact_chunk(A_hi[:, p0:p1], A_lo[:, p0:p1], B_hi[p0:p1], B_lo[p0:p1])
        X = part if X is None else X + part  # Python integers: exact
    return X


def _exact_chunk(A_hi, A_lo, B_hi, B_lo):
    """exact_product for k <= MAX_K"""
    m, k = A_hi.shape
    n = B_hi.shape[1]
    if k > MAX_K:
        raise ValueError("exact_fixed: k > 1024 (digit GEMMs would not be exact)")
    ea = _row_scale(A_hi)                       # rows of A
    eb = _row_scale(np.ascontiguousarray(B_hi.T))  # columns of B
    As_hi, As_lo = np.ldexp(A_hi, -ea[:, None]), np.ldexp(A_lo, -ea[:, None])
    Bs_hi, Bs_lo = np.ldexp(B_hi, -eb[None, :]), np.ldexp(B_lo, -eb[None, :])
    for sc, orig, e in ((As_hi, A_hi, ea[:, None]), (As_lo, A_lo, ea[:, None]),
                        (Bs_hi, B_hi, eb[None, :]), (Bs_lo, B_lo, eb[None, :])):
        if np.any(np.ldexp(sc, e) != orig):
            raise ValueError("exact_fixed: the scaling lost bits (subnormal limbs)")
    nda = _needed_digits(As_hi, As_lo)
    ndb = _needed_digits(Bs_hi, Bs_lo)
    da = [h + l for h, l in zip(_digits(As_hi, nda), _digits(As_lo, nda))]
    db = [h + l for h, l in zip(_digits(Bs_hi, ndb), _digits(Bs_lo, ndb))]
    ndiag = nda + ndb - 1
    diag = [np.zeros((m, n), dtype=np.int64) for _ in range(ndiag)]
    for s in range(nda):
        for t in range(ndb):
            p = da[s] @ db[t]           # exact integer-valued float64 GEMM
            diag[s + t] += p.astype(np.int64)
    # value = sum_d diag_d 2^(-20 (d + 2)) * 2^(ea_i + eb_j), in units 2^UNIT_EXP
    X = np.zeros((m, n), dtype=object)
    for d in range(ndiag):
        X = X * (1 << DIGIT) + diag[d].astype(object)
    # X is now in units 2^(-20 (ndiag + 1)); shift to 2^UNIT_EXP with the scales
    base = -DIGIT * (ndiag + 1)
    sh = (ea[:, None] + eb[None, :]) + base - UNIT_EXP
    if np.any(sh < 0):
        raise ValueError("exact_fixed: result below the unit grid")
    shifts = sh.astype(object)
    return np.frompyfunc(lambda x, s: x << s, 2, 1)(X, shifts)


def to_units(x):
    """binary64 array -> object array of exact integers in units 2^UNIT_EXP"""
    m, e = np.frexp(x)
    mi = np.ldexp(m, 53).astype(np.int64)  # exact: 53-bit integer mantissa
    sh = (e.astype(np.int64) - 53 - UNIT_EXP)
    f = np.frompyfunc(lambda a, s: (a << s) if s >= 0 else _exact_shr(a, s), 2, 1)
    return f(mi.astype(object), sh.astype(object))


def _exact_shr(a, s):
    if a % (1 << -s):
        raise ValueError("exact_fixed: value below the unit grid")
    return a >> -s


def errors(A_hi, A_lo, B_hi, B_lo, C_hi, C_lo):
    """err = (C_hi + C_lo) - C* exactly, returned as float64 (one rounding), and
    |C*| as float64, for every entry."""
    X = exact_product(A_hi, A_lo, B_hi, B_lo)
    C = to_units(C_hi) + to_units(C_lo)
    diff = C - X
    den = 1 << -UNIT_EXP
    tof = np.frompyfunc(lambda v: v / den, 1, 1)  # int / int: correctly rounded
    return tof(diff).astype(np.float64), np.abs(tof(X).astype(np.float64))
