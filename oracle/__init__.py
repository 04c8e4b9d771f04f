"""CPU ORACLE for the cascaded FP64x2 GEMM (arXiv 2303.04353).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2303_04353_b200``) never imports it, and the two share
no code: this wraps ``oracle/casc_oracle.c`` (plain C, binary64 RNE,
-ffp-contract=off) through ctypes.

Functions cite the PAPER.md passage they follow; see casc_oracle.c for the
step-by-step arithmetic and DESIGN.md §3/§4 for the readings and pins.
Parity unpinned: none.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "casc_oracle.c")
_SRC_I8 = os.path.join(_HERE, "casc_i8_oracle.c")  # NEXT-3: the INT8 cascade
_LIB = os.path.join(_HERE, "liboracle.so")
KC = 256

CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
          "-fopenmp", "-Wall"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (building the checker is not using it)."""
    stale = not os.path.exists(_LIB) or any(
        os.path.getmtime(_LIB) < os.path.getmtime(s) for s in (_SRC, _SRC_I8))
    if force or stale:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, _SRC_I8, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _setup(_lib)
    return _lib


_d = ctypes.c_double
_i64 = ctypes.c_int64
_pd = ctypes.POINTER(ctypes.c_double)
_pi32 = ctypes.POINTER(ctypes.c_int32)
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pu8 = ctypes.POINTER(ctypes.c_uint8)
_pint = ctypes.POINTER(ctypes.c_int)


def _side(side):
    return 0 if side in ("L", "l", 0) else 1


def casc_symm(side, uplo, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, nthreads: int = 0):
    """NEXT-4 SYMM (reading R28): C := alpha A B + beta C (side 'L') or alpha B A
    + beta C ('R'), A symmetric from its `uplo` triangle.  Returns new
    (C_hi, C_lo, flags)."""
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    m, n = C_hi.shape
    flags = np.zeros((m, n), dtype=np.uint8)
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    lib().orc_casc_symm(_side(side), lo_, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                        max(A_hi.shape[1], 1), _p(B_hi), _p(B_lo), max(n, 1), beta[0], beta[1],
                        _p(C_hi), _p(C_lo), max(n, 1), _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


def casc_trmm(side, uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", nthreads: int = 0):
    """NEXT-4 TRMM (reading R28): B := alpha op(A) B ('L') or alpha B op(A)
    ('R'), A triangular.  Returns new (B_hi, B_lo)."""
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    X_hi, X_lo = _c64(B_hi).copy(), _c64(B_lo).copy()
    m, n = X_hi.shape
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    tr = 1 if trans in ("T", "t", 1, True) else 0
    dg = 1 if diag in ("U", "u", 1, True) else 0
    lib().orc_casc_trmm(_side(side), lo_, tr, dg, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                        max(A_hi.shape[1], 1), _p(X_hi), _p(X_lo), max(n, 1), nthreads)
    return X_hi, X_lo


def casc_trsm_right(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", nthreads: int = 0):
    """NEXT-4 right-side TRSM (reading R29): X op(A) = alpha B, A n x n
    triangular, via the left TRSM on the transposes.  Returns new (X_hi, X_lo)."""
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    X_hi, X_lo = _c64(B_hi).copy(), _c64(B_lo).copy()
    m, n = X_hi.shape
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    tr = 1 if trans in ("T", "t", 1, True) else 0
    dg = 1 if diag in ("U", "u", 1, True) else 0
    lib().orc_casc_trsm_right(lo_, tr, dg, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                              max(n, 1), _p(X_hi), _p(X_lo), max(n, 1), nthreads)
    return X_hi, X_lo


def dd_trsm_plain(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N"):
    """Plain (unblocked) FP64x2 substitution for op(A) X = alpha B: the
    reference for the blocked casc_trsm (no shared block sizes)."""
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    tr = 1 if trans in ("T", "t", 1, True) else 0
    dg = 1 if diag in ("U", "u", 1, True) else 0
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    X_hi, X_lo = _c64(B_hi).copy(), _c64(B_lo).copy()
    m, n = X_hi.shape
    lib().orc_dd_trsm_plain(lo_, tr, dg, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo), max(m, 1),
                            _p(X_hi), _p(X_lo), max(n, 1))
    return X_hi, X_lo


def _setup(L):
    L.orc_two_sum.argtypes = [_d, _d, _pd, _pd]
    L.orc_fast_two_sum.argtypes = [_d, _d, _pd, _pd]
    L.orc_two_prod.argtypes = [_d, _d, _pd, _pd]
    L.orc_dd_add_d.argtypes = [_d, _d, _d, _pd, _pd]
    L.orc_dd_add.argtypes = [_d, _d, _d, _d, _pd, _pd]
    L.orc_dd_mul.argtypes = [_d, _d, _d, _d, _pd, _pd]
    L.orc_select_widths.argtypes = [_i64, _pint]
    L.orc_scale_exponent.argtypes = [_pd, _i64, _i64]
    L.orc_scale_exponent.restype = ctypes.c_int
    L.orc_split_scalar.argtypes = [_d, _d, ctypes.c_int, _pint, _pd]
    L.orc_split_a_panel.argtypes = [_i64, _i64, _pd, _pd, _i64, _pint, _pd, _pi32]
    L.orc_split_b_panel.argtypes = [_i64, _i64, _pd, _pd, _i64, _pint, _pd, _pi32]
    L.orc_panel_bins.argtypes = [_i64, _i64, _i64, _pd, _pd, _pint, _pd]
    L.orc_combine.argtypes = [_d, _d, _d, _d, ctypes.c_int, _pint, _pd, _pd]
    L.orc_casc_gemm.argtypes = [_i64, _i64, _i64, _pd, _pd, _i64, _pd, _pd, _i64, _pd, _pd,
                                _i64, _pu8, ctypes.c_int]
    L.orc_casc_gemm_ex.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, _d, _d, _pd,
                                   _pd, _i64, _pd, _pd, _i64, _d, _d, _pd, _pd, _i64, _pu8,
                                   ctypes.c_int]
    L.orc_casc_syrk.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d, _pd, _pd, _i64,
                                _d, _d, _pd, _pd, _i64, _pu8, ctypes.c_int]
    L.orc_dd_div.argtypes = [_d, _d, _d, _d, _pd, _pd]
    L.orc_trsm_diag_inv.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _pd, _pd, _i64, _pd, _pd]
    L.orc_casc_trsm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d, _pd,
                                _pd, _i64, _pd, _pd, _i64, ctypes.c_int]
    L.orc_casc_syr2k.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d, _pd, _pd, _i64,
                                 _pd, _pd, _i64, _d, _d, _pd, _pd, _i64, _pu8, ctypes.c_int]
    L.orc_casc_symm.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d, _pd, _pd, _i64,
                                _pd, _pd, _i64, _d, _d, _pd, _pd, _i64, _pu8, ctypes.c_int]
    L.orc_casc_trmm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64,
                                _i64, _d, _d, _pd, _pd, _i64, _pd, _pd, _i64, ctypes.c_int]
    L.orc_casc_trsm_right.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, _d,
                                      _d, _pd, _pd, _i64, _pd, _pd, _i64, ctypes.c_int]
    L.orc_dd_trsm_plain.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, _d,
                                    _d, _pd, _pd, _i64, _pd, _pd, _i64]
    L.orc_dd_gemm.argtypes = [_i64, _i64, _i64, _pd, _pd, _i64, _pd, _pd, _i64, _pd, _pd,
                              _i64, ctypes.c_int]
    L.orc_exact_entries.argtypes = [_i64, _pd, _pd, _i64, _pd, _pd, _i64, _i64, _pi64, _pi64,
                                    _pd, _pd, _i64, _pd, _pd, _pd, _pd, ctypes.c_int]
    L.orc_exact_sum.argtypes = [_i64, _pd, _pd, _pd]
    L.orc_exact_dot.argtypes = [_i64, _pd, _pd, _pd, _pd]
    L.orc_num_threads.restype = ctypes.c_int
    _pi8 = ctypes.POINTER(ctypes.c_int8)
    L.orc_i8_panel.restype = ctypes.c_int
    L.orc_i8_split_scalar.argtypes = [_d, _d, ctypes.c_int, ctypes.c_int, _pi8]
    L.orc_i8_split_rows.argtypes = [_i64, _i64, _pd, _pd, _i64, _i64, ctypes.c_int, _pi8, _pi32]
    L.orc_i8_panel_bins.argtypes = [_i64, _i64, _i64, ctypes.c_int, _pi8, _pi8, ctypes.c_int,
                                    _pi64]
    L.orc_i8_group_value.argtypes = [_pi64, ctypes.c_int, _pd, _pd]
    L.orc_i8_panel_value.argtypes = [_pi64, ctypes.c_int, ctypes.c_int, _pd, _pd]
    L.orc_i8_casc_gemm.argtypes = [_i64, _i64, _i64, _pd, _pd, _i64, _pd, _pd, _i64,
                                   ctypes.c_int, _pd, _pd, _i64, _pu8, ctypes.c_int]
    L.orc_i8_casc_gemm_ex.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, _d, _d,
                                      _pd, _pd, _i64, _pd, _pd, _i64, _d, _d, _pd, _pd, _i64,
                                      _pu8, ctypes.c_int, ctypes.c_int]
    L.orc_i8_casc_syrk.argtypes = [ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d, _pd, _pd, _i64,
                                   _d, _d, _pd, _pd, _i64, _pu8, ctypes.c_int, ctypes.c_int]
    L.orc_i8_casc_trsm.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, _d, _d,
                                   _pd, _pd, _i64, _pd, _pd, _i64, ctypes.c_int, ctypes.c_int]


def _p(a, ptr=_pd):
    return a.ctypes.data_as(ptr) if a is not None else None


def _c64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def num_threads() -> int:
    return lib().orc_num_threads()


# ---------------------------------------------------------------- DD primitives
def _pair(fn, *args):
    r1, r2 = _d(), _d()
    fn(*args, ctypes.byref(r1), ctypes.byref(r2))
    return r1.value, r2.value


def two_sum(a, b):
    """Knuth TwoSum (P:L756, P:L947 cite Dekker1971)."""
    return _pair(lib().orc_two_sum, a, b)


def fast_two_sum(a, b):
    return _pair(lib().orc_fast_two_sum, a, b)


def two_prod(a, b):
    """FMA TwoProd."""
    return _pair(lib().orc_two_prod, a, b)


def dd_add_d(th, tl, x):
    return _pair(lib().orc_dd_add_d, th, tl, x)


def dd_add(xh, xl, yh, yl):
    return _pair(lib().orc_dd_add, xh, xl, yh, yl)


def dd_mul(xh, xl, yh, yl):
    return _pair(lib().orc_dd_mul, xh, xl, yh, yl)


# ---------------------------------------------------------------- cascade steps
def select_widths(k: int):
    """(c0, c1, c2) from the §3.3 bit budgets with k_eff = min(k, 256)."""
    c = (ctypes.c_int * 3)()
    lib().orc_select_widths(k, c)
    return tuple(c)


def _cw(k):
    c = (ctypes.c_int * 3)(*select_widths(k))
    return c


def scale_exponent(hi: np.ndarray) -> int:
    """e with max|hi| in [2^(e-1), 2^e); 0 for all zeros."""
    hi = _c64(hi).ravel()
    return lib().orc_scale_exponent(_p(hi), hi.size, 1)


def split_scalar(hi: float, lo: float, e: int, widths):
    """Appendix A split of one FP64x2 value -> (chi0..chi3)."""
    c = (ctypes.c_int * 3)(*widths)
    out = (ctypes.c_double * 4)()
    lib().orc_split_scalar(hi, lo, e, c, out)
    return tuple(out)


def split_a_panel(A_hi, A_lo, widths=None):
    """Split an m x kp panel of A conformally per row (§3.4, App. A).
    Returns slices (4, m, kp) in the paper's normalisation and e (m,)."""
    A_hi, A_lo = _c64(A_hi), _c64(A_lo)
    m, kp = A_hi.shape
    c = (ctypes.c_int * 3)(*(widths or select_widths(kp)))
    S = np.empty((4, m, kp))
    e = np.empty(m, dtype=np.int32)
    lib().orc_split_a_panel(m, kp, _p(A_hi), _p(A_lo), kp, c, _p(S), _p(e, _pi32))
    return S, e


def split_b_panel(B_hi, B_lo, widths=None):
    """Split a kp x n panel of B conformally per column, plus B4, B5, B6
    (P:L1403-1404).  Returns slices (7, kp, n) and f (n,)."""
    B_hi, B_lo = _c64(B_hi), _c64(B_lo)
    kp, n = B_hi.shape
    c = (ctypes.c_int * 3)(*(widths or select_widths(kp)))
    S = np.empty((7, kp, n))
    f = np.empty(n, dtype=np.int32)
    lib().orc_split_b_panel(kp, n, _p(B_hi), _p(B_lo), n, c, _p(S), _p(f, _pi32))
    return S, f


def panel_bins(SA, SB, widths):
    """Bins 0, 1, 2, 3-6 of one panel (eqn:Gemm10)."""
    SA, SB = _c64(SA), _c64(SB)
    _, m, kp = SA.shape
    n = SB.shape[2]
    c = (ctypes.c_int * 3)(*widths)
    bins = np.empty((4, m, n))
    lib().orc_panel_bins(m, n, kp, _p(SA), _p(SB), c, _p(bins))
    return bins


def combine(bin0, bin1, bin2, bin36, escale, widths):
    """fl_casc of one element -> (t_hi, t_lo)."""
    c = (ctypes.c_int * 3)(*widths)
    r1, r2 = _d(), _d()
    lib().orc_combine(bin0, bin1, bin2, bin36, int(escale), c, ctypes.byref(r1),
                      ctypes.byref(r2))
    return r1.value, r2.value


def casc_gemm(A_hi, A_lo, B_hi, B_lo, nthreads: int = 0):
    """ORACLE-CASCADE: C := A B through ten cascading FP64 GEMMs per k_C panel.
    Returns (C_hi, C_lo, flags)."""
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    m, k = A_hi.shape
    n = B_hi.shape[1]
    C_hi = np.empty((m, n))
    C_lo = np.empty((m, n))
    flags = np.empty((m, n), dtype=np.uint8)
    lib().orc_casc_gemm(m, n, k, _p(A_hi), _p(A_lo), k, _p(B_hi), _p(B_lo), n, _p(C_hi),
                        _p(C_lo), n, _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


def casc_gemm_ex(transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo,
                 nthreads: int = 0):
    """NEXT-4: C := alpha (x) op(A) op(B) (+) beta (x) C (reading R21).  A, B
    are the STORED matrices (A is k x m when transa); alpha, beta (hi, lo).
    Returns new (C_hi, C_lo, flags)."""
    ta, tb = int(transa in ("T", 1, True)), int(transb in ("T", 1, True))
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    m, n = C_hi.shape
    k = A_hi.shape[0] if ta else A_hi.shape[1]
    flags = np.zeros((m, n), dtype=np.uint8)
    lib().orc_casc_gemm_ex(ta, tb, m, n, k, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                           A_hi.shape[1] if A_hi.size else 1, _p(B_hi), _p(B_lo),
                           B_hi.shape[1] if B_hi.size else 1, beta[0], beta[1], _p(C_hi),
                           _p(C_lo), n, _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


def casc_syrk(uplo, trans, alpha, A_hi, A_lo, beta, C_hi, C_lo, flags=None, nthreads: int = 0):
    """NEXT-4 SYRK: the lower ('L') / upper ('U') triangle of
    casc_gemm_ex(trans, not trans, alpha, A, A, beta, C); the other triangle
    of C and flags is returned unchanged.  A is the STORED matrix (n x k for
    trans 'N', k x n for 'T').  Returns new (C_hi, C_lo, flags)."""
    lo = 0 if uplo in ("L", "l", 0) else 1
    tr = int(trans in ("T", "t", 1, True))
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    n = C_hi.shape[0]
    k = A_hi.shape[0] if tr else A_hi.shape[1]
    flags = np.zeros((n, n), dtype=np.uint8) if flags is None else np.array(flags, np.uint8)
    lib().orc_casc_syrk(lo, tr, n, k, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                        A_hi.shape[1] if A_hi.size else 1, beta[0], beta[1], _p(C_hi), _p(C_lo),
                        n, _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


def casc_syr2k(uplo, trans, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, flags=None,
               nthreads: int = 0):
    """NEXT-4 SYR2K (reading R30): on the `uplo` triangle C := alpha op(A)
    op(B)^T + beta C, then C := alpha op(B) op(A)^T + C (cascaded GEMMs, R21);
    flags = OR of both.  A, B stored n x k ('N') or k x n ('T')."""
    lo = 0 if uplo in ("L", "l", 0) else 1
    tr = int(trans in ("T", "t", 1, True))
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    n = C_hi.shape[0]
    k = A_hi.shape[0] if tr else A_hi.shape[1]
    flags = np.zeros((n, n), dtype=np.uint8) if flags is None else np.array(flags, np.uint8)
    lib().orc_casc_syr2k(lo, tr, n, k, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                         A_hi.shape[1] if A_hi.size else 1, _p(B_hi), _p(B_lo),
                         B_hi.shape[1] if B_hi.size else 1, beta[0], beta[1], _p(C_hi), _p(C_lo),
                         n, _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


TRSM_NB = 256


def dd_div(xh, xl, yh, yl):
    """FP64x2 long division (reading R27)."""
    return _pair(lib().orc_dd_div, xh, xl, yh, yl)


def trsm_diag_inv(uplo, diag, A_hi, A_lo):
    """Inverses of the TRSM_NB diagonal blocks of the triangular A (R27):
    (nblk, TRSM_NB, TRSM_NB) hi and lo arrays."""
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    dg = 1 if diag in ("U", "u", 1, True) else 0
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    m = A_hi.shape[0]
    nblk = -(-m // TRSM_NB)
    Ih = np.zeros((nblk, TRSM_NB, TRSM_NB))
    Il = np.zeros((nblk, TRSM_NB, TRSM_NB))
    lib().orc_trsm_diag_inv(lo_, dg, m, _p(A_hi), _p(A_lo), m, _p(Ih), _p(Il))
    return Ih, Il


def casc_trsm(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", nthreads: int = 0):
    """NEXT-4 TRSM (reading R27): X with op(A) X = alpha B, left side, op(A) = A
    or A^T; A m x m triangular; returns new (X_hi, X_lo)."""
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    tr = 1 if trans in ("T", "t", 1, True) else 0
    dg = 1 if diag in ("U", "u", 1, True) else 0
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    X_hi, X_lo = _c64(B_hi).copy(), _c64(B_lo).copy()
    m, n = X_hi.shape
    lib().orc_casc_trsm(lo_, tr, dg, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo), max(m, 1),
                        _p(X_hi), _p(X_lo), max(n, 1), nthreads)
    return X_hi, X_lo


def dd_gemm(A_hi, A_lo, B_hi, B_lo, nthreads: int = 0):
    """ORACLE-DD: triple-loop FP64x2 GEMM."""
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    m, k = A_hi.shape
    n = B_hi.shape[1]
    C_hi = np.empty((m, n))
    C_lo = np.empty((m, n))
    lib().orc_dd_gemm(m, n, k, _p(A_hi), _p(A_lo), k, _p(B_hi), _p(B_lo), n, _p(C_hi),
                      _p(C_lo), n, nthreads)
    return C_hi, C_lo


def exact_entries(A_hi, A_lo, B_hi, B_lo, ii, jj, C_hi=None, C_lo=None, nthreads: int = 0):
    """ORACLE-EXACT for entries (ii[t], jj[t]): exact C* as RN double-double,
    err = RN((C_hi + C_lo) - C*) if C given, and |A||B| rounded.
    Returns dict(ex_hi, ex_lo, err, absab)."""
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    m, k = A_hi.shape
    n = B_hi.shape[1]
    ii = np.ascontiguousarray(ii, dtype=np.int64)
    jj = np.ascontiguousarray(jj, dtype=np.int64)
    T = ii.size
    ex_hi, ex_lo, absab = np.empty(T), np.empty(T), np.empty(T)
    err = np.empty(T) if C_hi is not None else None
    if C_hi is not None:
        C_hi, C_lo = _c64(C_hi), _c64(C_lo)
        ldc = C_hi.shape[1]
    else:
        ldc = 0
    lib().orc_exact_entries(k, _p(A_hi), _p(A_lo), k, _p(B_hi), _p(B_lo), n, T,
                            _p(ii, _pi64), _p(jj, _pi64), _p(C_hi), _p(C_lo), ldc, _p(ex_hi),
                            _p(ex_lo), _p(err), _p(absab), nthreads)
    return dict(ex_hi=ex_hi, ex_lo=ex_lo, err=err, absab=absab)


def exact_sum(x):
    x = _c64(x).ravel()
    return _pair(lib().orc_exact_sum, x.size, _p(x))


def exact_dot(x, y):
    x, y = _c64(x).ravel(), _c64(y).ravel()
    return _pair(lib().orc_exact_dot, x.size, _p(x), _p(y))


def north_star_bound(k: int, absab):
    """|C_gpu - C*| <= 4 k 2^-104 (|A||B|)_ij (BASELINE.json north_star)."""
    return 4.0 * k * 2.0 ** -104 * np.asarray(absab)


def cascerr_bound(k: int, absab, normx, normy, widths):
    """eq:cascerr: |x|^T|y| eps_hat + 40 k^2 eps_tilde ||x|| ||y||,
    eps_hat = 2^-106, eps_tilde = 2^-(D2 + 53)."""
    D2 = sum(widths)
    return (np.asarray(absab) * 2.0 ** -106
            + 40.0 * k * k * 2.0 ** -(D2 + 53) * np.asarray(normx) * np.asarray(normy))


# ---------------------------------------------------------------- NEXT-3: INT8 cascade
# (casc_i8_oracle.c; readings R22-R26 in DESIGN.md §3)
_pi8 = ctypes.POINTER(ctypes.c_int8)


def i8_panel() -> int:
    """k_C8, the INT8 cascade's panel depth (reading R22)."""
    return lib().orc_i8_panel()


def i8_split_scalar(hi: float, lo: float, e: int, y: int):
    """The y balanced base-256 int8 slices of one FP64x2 value (reading R23)."""
    d = (ctypes.c_int8 * y)()
    lib().orc_i8_split_scalar(hi, lo, int(e), int(y), d)
    return tuple(d)


def i8_split_a_panel(A_hi, A_lo, y: int):
    """Slices of an m x kp panel of A per row -> (D (y, m, kp) int8, e (m,))."""
    A_hi, A_lo = _c64(A_hi), _c64(A_lo)
    m, kp = A_hi.shape
    D = np.empty((y, m, kp), dtype=np.int8)
    e = np.empty(m, dtype=np.int32)
    lib().orc_i8_split_rows(m, kp, _p(A_hi), _p(A_lo), kp, 1, y, _p(D, _pi8), _p(e, _pi32))
    return D, e


def i8_split_b_panel(B_hi, B_lo, y: int):
    """Slices of a kp x n panel of B per column -> (D (y, n, kp) int8, f (n,))."""
    B_hi, B_lo = _c64(B_hi), _c64(B_lo)
    kp, n = B_hi.shape
    D = np.empty((y, n, kp), dtype=np.int8)
    f = np.empty(n, dtype=np.int32)
    lib().orc_i8_split_rows(n, kp, _p(B_hi), _p(B_lo), 1, n, y, _p(D, _pi8), _p(f, _pi32))
    return D, f


def i8_panel_bins(DA, DB, nbins: int | None = None):
    """Exact bins of one panel (reading R24): bin_s = sum over i + j = s of
    DA_i DB_j^T, s < nbins (default y: the paper's triangle)."""
    DA = np.ascontiguousarray(DA, dtype=np.int8)
    DB = np.ascontiguousarray(DB, dtype=np.int8)
    y, m, kp = DA.shape
    n = DB.shape[1]
    nb = y if nbins is None else nbins
    bins = np.empty((nb, m, n), dtype=np.int64)
    lib().orc_i8_panel_bins(m, n, kp, y, _p(DA, _pi8), _p(DB, _pi8), nb, _p(bins, _pi64))
    return bins


def i8_group_value(b):
    """Exact FP64x2 value of up to four consecutive bins (reading R25)."""
    b = np.ascontiguousarray(b, dtype=np.int64)
    return _pair(lib().orc_i8_group_value, _p(b, _pi64), b.size)


def i8_panel_value(b, w0: int):
    """Panel value T of one element (reading R25, rev. 2): the FP64x2 number
    nearest x = sum_s b[s] 2^(w0 + 8(y-1-s)), y = len(b)."""
    b = np.ascontiguousarray(b, dtype=np.int64)
    return _pair(lib().orc_i8_panel_value, _p(b, _pi64), b.size, int(w0))


def i8_casc_syrk(uplo, trans, alpha, A_hi, A_lo, beta, C_hi, C_lo, flags=None, y: int = 14,
                 nthreads: int = 0):
    """NEXT-4 SYRK on the INT8 cascade: the triangle of i8_casc_gemm_ex(trans,
    not trans, alpha, A, A, beta, C); other triangle and its flags unchanged."""
    lo = 0 if uplo in ("L", "l", 0) else 1
    tr = int(trans in ("T", "t", 1, True))
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    n = C_hi.shape[0]
    k = A_hi.shape[0] if tr else A_hi.shape[1]
    flags = np.zeros((n, n), dtype=np.uint8) if flags is None else np.array(flags, np.uint8)
    lib().orc_i8_casc_syrk(lo, tr, n, k, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                           A_hi.shape[1] if A_hi.size else 1, beta[0], beta[1], _p(C_hi),
                           _p(C_lo), n, _p(flags, _pu8), int(y), nthreads)
    return C_hi, C_lo, flags


def i8_casc_trsm(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", y: int = 14,
                 nthreads: int = 0):
    """NEXT-4 TRSM on the INT8 cascade (reading R27): X with op(A) X = alpha B."""
    lo_ = 0 if uplo in ("L", "l", 0) else 1
    tr = 1 if trans in ("T", "t", 1, True) else 0
    dg = 1 if diag in ("U", "u", 1, True) else 0
    A_hi, A_lo = map(_c64, (A_hi, A_lo))
    X_hi, X_lo = _c64(B_hi).copy(), _c64(B_lo).copy()
    m, n = X_hi.shape
    lib().orc_i8_casc_trsm(lo_, tr, dg, m, n, alpha[0], alpha[1], _p(A_hi), _p(A_lo), max(m, 1),
                           _p(X_hi), _p(X_lo), max(n, 1), int(y), nthreads)
    return X_hi, X_lo


def i8_casc_gemm(A_hi, A_lo, B_hi, B_lo, y: int = 14, nthreads: int = 0):
    """ORACLE-I8CASCADE: C := A B through y int8 slices (NEXT-3).
    Returns (C_hi, C_lo, flags)."""
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    m, k = A_hi.shape
    n = B_hi.shape[1]
    C_hi = np.empty((m, n))
    C_lo = np.empty((m, n))
    flags = np.empty((m, n), dtype=np.uint8)
    lib().orc_i8_casc_gemm(m, n, k, _p(A_hi), _p(A_lo), k, _p(B_hi), _p(B_lo), n, int(y),
                           _p(C_hi), _p(C_lo), n, _p(flags, _pu8), nthreads)
    return C_hi, C_lo, flags


def i8_casc_gemm_ex(transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, y: int = 14,
                    nthreads: int = 0):
    """NEXT-4 on the INT8 cascade: C := alpha (x) op(A) op(B) (+) beta (x) C
    (reading R21).  A, B are the STORED matrices; alpha, beta (hi, lo).
    Returns new (C_hi, C_lo, flags)."""
    ta, tb = int(transa in ("T", 1, True)), int(transb in ("T", 1, True))
    A_hi, A_lo, B_hi, B_lo = map(_c64, (A_hi, A_lo, B_hi, B_lo))
    C_hi, C_lo = _c64(C_hi).copy(), _c64(C_lo).copy()
    m, n = C_hi.shape
    k = A_hi.shape[0] if ta else A_hi.shape[1]
    flags = np.zeros((m, n), dtype=np.uint8)
    lib().orc_i8_casc_gemm_ex(ta, tb, m, n, k, alpha[0], alpha[1], _p(A_hi), _p(A_lo),
                              A_hi.shape[1] if A_hi.size else 1, _p(B_hi), _p(B_lo),
                              B_hi.shape[1] if B_hi.size else 1, beta[0], beta[1], _p(C_hi),
                              _p(C_lo), n, _p(flags, _pu8), int(y), nthreads)
    return C_hi, C_lo, flags
