"""paper_2303_04353_b200 — B200-native cascaded FP64x2 GEMM (arXiv 2303.04353).

Thin Python binding over the C ABI of ``libcasc.so`` (include/casc.h).  Every
function here has the name of the C entry point it marshals to and does
argument marshalling only (pointers, leading dimensions, the current CUDA
stream); every step of the method runs in the library's sm_100a kernels.
PyTorch is used for device memory and streams only.

There is no CPU fallback: importing this package fails loudly if the CUDA
library has not been built (``python -c "import __graft_entry__ as g; g.build()"``).
"""

from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CASC_LIB_PATH") or os.path.join(_HERE, "libcasc.so")
KC = 256

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build the CUDA extension first "
                      "(__graft_entry__.build()); there is no CPU fallback")
_lib = ctypes.CDLL(LIB_PATH)

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_sz = ctypes.c_size_t


def _sig(name, args, res=ctypes.c_int):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = res
    return f


_sig("casc_status_string", [ctypes.c_int], ctypes.c_char_p)
_sig("casc_select_widths", [_i64, ctypes.POINTER(ctypes.c_int)])
_sig("casc_gemm_fp64x2", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp,
                          _vp])
_sig("casc_gemm_fp64x2_ws", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                             _vp, _vp, _sz, _vp])
_sig("casc_workspace_bytes", [_i64, _i64, _i64], _sz)
_sig("casc_finalize", [])
_sig("casc_packed_a_bytes", [_i64, _i64], _sz)
_sig("casc_packed_b_bytes", [_i64, _i64], _sz)
_sig("casc_packed_a_block_bytes", [_i64], _sz)
_sig("casc_packed_b_block_bytes", [_i64], _sz)
_sig("casc_pack_a", [_i64, _i64, _vp, _vp, _i64, _vp, _vp])
_sig("casc_pack_b", [_i64, _i64, _vp, _vp, _i64, _vp, _vp])
_sig("casc_gemm_packed", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp])
_sig("casc_gemm_packed_ld", [_i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _vp])
_sig("casc_split_a", [_i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp])
_sig("casc_split_b", [_i64, _i64, _vp, _vp, _i64, _vp, _vp, _vp])
_sig("casc_debug_bins", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _i64, _vp, _vp])
_sig("casc_last_launch_count", [])
_sig("casc_debug_ldexp", [_i64, _vp, _vp, _vp, _vp])
_sig("casc_gemm_fp64x2_simple", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                                 _i64, _vp, _vp])
_sig("casc_slice_product", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_int,
                            ctypes.c_int, _i64, _vp, _vp])

EXPORTED = ["casc_status_string", "casc_select_widths", "casc_gemm_fp64x2",
            "casc_gemm_fp64x2_ws", "casc_workspace_bytes", "casc_finalize",
            "casc_packed_a_bytes", "casc_packed_b_bytes", "casc_packed_a_block_bytes",
            "casc_packed_b_block_bytes", "casc_pack_a", "casc_pack_b", "casc_gemm_packed",
            "casc_split_a", "casc_split_b", "casc_debug_bins", "casc_last_launch_count",
            "casc_gemm_fp64x2_simple", "casc_slice_product", "casc_gemm_fp64x2_ex",
            "casc_i8_gemm_fp64x2", "casc_i8_gemm_fp64x2_ws", "casc_i8_workspace_bytes",
            "casc_i8_packed_bytes", "casc_i8_finalize", "casc_i8_split", "casc_i8_debug_bins",
            "casc_i8_packed_block_bytes", "casc_i8_pack", "casc_i8_gemm_ws_bytes",
            "casc_i8_gemm_packed", "casc_i8_gemm_fp64x2_ex", "casc_gemm_fp64x2_host",
            "casc_i8_gemm_fp64x2_host", "casc_syrk_fp64x2", "casc_trsm_fp64x2",
            "casc_trsm_diag_inv", "casc_i8_syrk_fp64x2", "casc_i8_trsm_fp64x2",
            "casc_debug_ldexp", "casc_gemm_packed_ld", "casc_i8_gemm_packed_ld",
            "casc_symm_fp64x2", "casc_trmm_fp64x2", "casc_trsm_fp64x2_right",
            "casc_syr2k_fp64x2"]

_sig("casc_i8_gemm_fp64x2", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                             _vp, ctypes.c_int, _vp])
_sig("casc_i8_gemm_fp64x2_ws", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                                _i64, _vp, ctypes.c_int, _vp, _sz, _vp])
_sig("casc_i8_workspace_bytes", [_i64, _i64, _i64, ctypes.c_int], _sz)
_sig("casc_i8_packed_bytes", [_i64, _i64, ctypes.c_int], _sz)
_sig("casc_i8_finalize", [])
_sig("casc_i8_split", [_i64, _i64, _vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp])
_sig("casc_i8_debug_bins", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_int,
                            _i64, _vp, _vp])
_sig("casc_i8_packed_block_bytes", [_i64, ctypes.c_int], _sz)
_sig("casc_i8_pack", [_i64, _i64, _vp, _vp, _i64, ctypes.c_int, ctypes.c_int, _vp, _vp])
_sig("casc_i8_gemm_ws_bytes", [_i64, _i64], _sz)
_sig("casc_i8_gemm_packed", [_i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _i64, _vp, _vp,
                             _sz, _vp])
_sig("casc_i8_gemm_packed_ld", [_i64, _i64, _i64, ctypes.c_int, _vp, _vp, _vp, _vp, _i64, _vp,
                                  _i64, _vp, _sz, _vp])
I8_KC = 8192
I8_DEFAULT_SLICES = 14

_sig("casc_gemm_fp64x2_ex", [ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, ctypes.c_double,
                             ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_double,
                             ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _sz, _vp])
CASC_OP_N, CASC_OP_T = 0, 1
CASC_LOWER, CASC_UPPER = 0, 1
CASC_NONUNIT, CASC_UNIT = 0, 1
TRSM_NB = 256
_sig("casc_trsm_fp64x2", [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_double,
                          ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, _vp])
_sig("casc_trsm_diag_inv", [ctypes.c_int, ctypes.c_int, _i64, _vp, _vp, _i64, _vp, _vp, _vp])


def _uplo_diag(uplo, diag):
    if uplo not in ("L", "l", "U", "u", 0, 1):
        raise ValueError("uplo must be 'L' or 'U'")
    if diag not in ("N", "n", "U", "u", 0, 1):
        raise ValueError("diag must be 'N' or 'U'")
    return (CASC_LOWER if uplo in ("L", "l", 0) else CASC_UPPER,
            CASC_UNIT if diag in ("U", "u", 1) else CASC_NONUNIT)


_sig("casc_i8_syrk_fp64x2", [ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_double,
                             ctypes.c_double, _vp, _vp, _i64, ctypes.c_double, ctypes.c_double, _vp,
                             _vp, _i64, _vp, ctypes.c_int, _vp])


def casc_i8_syrk_fp64x2(uplo, trans, alpha, A_hi, A_lo, beta, C_hi, C_lo, flags=None, y: int = 14,
                        stream=None):
    """casc_syrk_fp64x2 on the INT8 cascade (NEXT-3 + NEXT-4)."""
    lo, _ = _uplo_diag(uplo, "N")
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = (alpha, 0.0) if isinstance(alpha, (int, float)) else alpha
    bh, bl = (beta, 0.0) if isinstance(beta, (int, float)) else beta
    n = C_hi.shape[0]
    ldc = _ld_pair(C_hi, C_lo, "C")
    if A_hi is None:
        lda, k = 1, 0
    else:
        lda = _ld_pair(A_hi, A_lo, "A")
        k = A_hi.shape[0] if tr else A_hi.shape[1]
    if flags is not None and (flags.dtype != torch.uint8 or tuple(flags.shape) != (n, n)):
        raise TypeError("flags must be a contiguous (n, n) uint8 CUDA tensor")
    _check(_lib.casc_i8_syrk_fp64x2(lo, tr, n, k, float(ah), float(al), _ptr(A_hi), _ptr(A_lo),
                                    lda, float(bh), float(bl), _ptr(C_hi), _ptr(C_lo), ldc,
                                    _ptr(flags), int(y), _stream(stream)), "casc_i8_syrk_fp64x2")
    return C_hi, C_lo, flags


def casc_trsm_fp64x2(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", stream=None):
    """TRSM on the cascaded GEMM (NEXT-4, reading R27): solve op(A) X = alpha B
    (left side, op(A) = A or A^T), A m x m triangular; X overwrites B_hi / B_lo."""
    lo, dg = _uplo_diag(uplo, diag)
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = (alpha, 0.0) if isinstance(alpha, (int, float)) else alpha
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, n = B_hi.shape
    if tuple(A_hi.shape) != (m, m):
        raise ValueError("A must be m x m")
    _check(_lib.casc_trsm_fp64x2(lo, tr, dg, m, n, float(ah), float(al), _ptr(A_hi), _ptr(A_lo),
                                 lda, _ptr(B_hi), _ptr(B_lo), ldb, _stream(stream)),
           "casc_trsm_fp64x2")
    return B_hi, B_lo


_sig("casc_syr2k_fp64x2", [ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_double,
                           ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_double,
                           ctypes.c_double, _vp, _vp, _i64, _vp, _vp])


def casc_syr2k_fp64x2(uplo, trans, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, flags=None,
                      stream=None):
    """SYR2K on the cascaded GEMM (casc.h, reading R30): on the 'L' / 'U'
    triangle of the n x n C, C := alpha op(A) op(B)^T + alpha op(B) op(A)^T +
    beta C.  A, B stored n x k ('N') or k x n ('T'); A_hi None means k = 0."""
    lo = CASC_LOWER if uplo in ("L", "l", 0) else CASC_UPPER
    if uplo not in ("L", "l", "U", "u", 0, 1):
        raise ValueError("uplo must be 'L' or 'U'")
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = _dd(alpha)
    bh, bl = _dd(beta)
    n = C_hi.shape[0]
    ldc = _ld_pair(C_hi, C_lo, "C")
    if A_hi is None:
        lda = ldb = 1
        k = 0
    else:
        lda = _ld_pair(A_hi, A_lo, "A")
        ldb = _ld_pair(B_hi, B_lo, "B")
        k = A_hi.shape[0] if tr else A_hi.shape[1]
    if flags is not None and (flags.dtype != torch.uint8 or tuple(flags.shape) != (n, n)
                              or not flags.is_contiguous()):
        raise TypeError("flags must be a contiguous (n, n) uint8 CUDA tensor")
    _check(_lib.casc_syr2k_fp64x2(lo, tr, n, k, ah, al, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                  _ptr(B_lo), ldb, bh, bl, _ptr(C_hi), _ptr(C_lo), ldc,
                                  _ptr(flags), _stream(stream)), "casc_syr2k_fp64x2")
    return C_hi, C_lo, flags


_sig("casc_symm_fp64x2", [ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_double,
                          ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_double,
                          ctypes.c_double, _vp, _vp, _i64, _vp, _vp])
_sig("casc_trmm_fp64x2", [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64,
                          ctypes.c_double, ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, _vp])
_sig("casc_trsm_fp64x2_right", [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64,
                                ctypes.c_double, ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64,
                                _vp])
CASC_LEFT, CASC_RIGHT = 0, 1


def _side(side):
    if side not in ("L", "l", "R", "r", 0, 1):
        raise ValueError("side must be 'L' or 'R'")
    return CASC_LEFT if side in ("L", "l", 0) else CASC_RIGHT


def _dd(x):
    return (float(x), 0.0) if isinstance(x, (int, float)) else (float(x[0]), float(x[1]))


def casc_symm_fp64x2(side, uplo, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, flags=None,
                     stream=None):
    """SYMM on the cascaded GEMM (casc.h): C := alpha A B + beta C (side 'L') or
    alpha B A + beta C ('R'), A symmetric, only its `uplo` triangle read; C
    (m x n) updated in place.  A_hi None means alpha = 0 (A, B not read)."""
    sd = _side(side)
    lo, _ = _uplo_diag(uplo, "N")
    ah, al = _dd(alpha)
    bh, bl = _dd(beta)
    m, n = C_hi.shape
    ldc = _ld_pair(C_hi, C_lo, "C")
    lda = _ld_pair(A_hi, A_lo, "A") if A_hi is not None else 1
    ldb = _ld_pair(B_hi, B_lo, "B") if B_hi is not None else max(n, 1)
    if A_hi is None:
        ah = al = 0.0
    if flags is not None and (flags.dtype != torch.uint8 or tuple(flags.shape) != (m, n)
                              or not flags.is_contiguous()):
        raise TypeError("flags must be a contiguous (m, n) uint8 CUDA tensor")
    _check(_lib.casc_symm_fp64x2(sd, lo, m, n, ah, al, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                 _ptr(B_lo), ldb, bh, bl, _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags),
                                 _stream(stream)), "casc_symm_fp64x2")
    return C_hi, C_lo, flags


def casc_trmm_fp64x2(side, uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", stream=None):
    """TRMM on the cascaded GEMM: B := alpha op(A) B ('L') or alpha B op(A) ('R'),
    A triangular; B overwritten."""
    sd = _side(side)
    lo, dg = _uplo_diag(uplo, diag)
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = _dd(alpha)
    m, n = B_hi.shape
    _check(_lib.casc_trmm_fp64x2(sd, lo, tr, dg, m, n, ah, al, _ptr(A_hi), _ptr(A_lo),
                                 _ld_pair(A_hi, A_lo, "A"), _ptr(B_hi), _ptr(B_lo),
                                 _ld_pair(B_hi, B_lo, "B"), _stream(stream)), "casc_trmm_fp64x2")
    return B_hi, B_lo


def casc_trsm_fp64x2_right(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", stream=None):
    """Right-side TRSM: solve X op(A) = alpha B (A n x n triangular, B m x n);
    X overwrites B."""
    lo, dg = _uplo_diag(uplo, diag)
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = _dd(alpha)
    m, n = B_hi.shape
    if tuple(A_hi.shape) != (n, n):
        raise ValueError("A must be n x n")
    _check(_lib.casc_trsm_fp64x2_right(lo, tr, dg, m, n, ah, al, _ptr(A_hi), _ptr(A_lo),
                                       _ld_pair(A_hi, A_lo, "A"), _ptr(B_hi), _ptr(B_lo),
                                       _ld_pair(B_hi, B_lo, "B"), _stream(stream)),
           "casc_trsm_fp64x2_right")
    return B_hi, B_lo


_sig("casc_i8_trsm_fp64x2", [ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64, _i64,
                             ctypes.c_double, ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64,
                             ctypes.c_int, _vp])


def casc_i8_trsm_fp64x2(uplo, diag, alpha, A_hi, A_lo, B_hi, B_lo, trans="N", y: int = 14,
                        stream=None):
    """casc_trsm_fp64x2 with the INT8 cascade as the GEMM (bit-exact with its oracle)."""
    lo, dg = _uplo_diag(uplo, diag)
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = (alpha, 0.0) if isinstance(alpha, (int, float)) else alpha
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, n = B_hi.shape
    if tuple(A_hi.shape) != (m, m):
        raise ValueError("A must be m x m")
    _check(_lib.casc_i8_trsm_fp64x2(lo, tr, dg, m, n, float(ah), float(al), _ptr(A_hi),
                                    _ptr(A_lo), lda, _ptr(B_hi), _ptr(B_lo), ldb, int(y),
                                    _stream(stream)), "casc_i8_trsm_fp64x2")
    return B_hi, B_lo


def casc_trsm_diag_inv(uplo, diag, A_hi, A_lo, stream=None):
    """The TRSM's inverted 256 x 256 diagonal blocks: (nblk, 256, 256) hi, lo."""
    lo, dg = _uplo_diag(uplo, diag)
    lda = _ld_pair(A_hi, A_lo, "A")
    m = A_hi.shape[0]
    nblk = -(-m // TRSM_NB)
    inv_hi = torch.empty((nblk, TRSM_NB, TRSM_NB), dtype=torch.float64, device=A_hi.device)
    inv_lo = torch.empty_like(inv_hi)
    _check(_lib.casc_trsm_diag_inv(lo, dg, m, _ptr(A_hi), _ptr(A_lo), lda, _ptr(inv_hi),
                                   _ptr(inv_lo), _stream(stream)), "casc_trsm_diag_inv")
    return inv_hi, inv_lo
_sig("casc_syrk_fp64x2", [ctypes.c_int, ctypes.c_int, _i64, _i64, ctypes.c_double, ctypes.c_double,
                          _vp, _vp, _i64, ctypes.c_double, ctypes.c_double, _vp, _vp, _i64, _vp,
                          _vp, _sz, _vp])


def casc_syrk_fp64x2(uplo, trans, alpha, A_hi, A_lo, beta, C_hi, C_lo, flags=None,
                     workspace=None, stream=None):
    """SYRK on the cascaded GEMM (NEXT-4, casc.h): C := alpha op(A) op(A)^T +
    beta C on the lower ('L') or upper ('U') triangle of the n x n C_hi / C_lo
    (updated in place, the other triangle untouched).  A is the stored matrix:
    n x k for trans 'N', k x n for 'T'; A_hi None means k = 0."""
    lo = CASC_LOWER if uplo in ("L", "l", 0) else CASC_UPPER
    if uplo not in ("L", "l", "U", "u", 0, 1):
        raise ValueError("uplo must be 'L' or 'U'")
    tr = 1 if trans in ("T", "t", 1, True) else 0
    ah, al = (alpha, 0.0) if isinstance(alpha, (int, float)) else alpha
    bh, bl = (beta, 0.0) if isinstance(beta, (int, float)) else beta
    n = C_hi.shape[0]
    ldc = _ld_pair(C_hi, C_lo, "C")
    if A_hi is None:
        lda, k = 1, 0
    else:
        lda = _ld_pair(A_hi, A_lo, "A")
        k = A_hi.shape[0] if tr else A_hi.shape[1]
    if flags is not None and (flags.dtype != torch.uint8 or tuple(flags.shape) != (n, n)):
        raise TypeError("flags must be a contiguous (n, n) uint8 CUDA tensor")
    _check(_lib.casc_syrk_fp64x2(lo, tr, n, k, float(ah), float(al), _ptr(A_hi), _ptr(A_lo), lda,
                                 float(bh), float(bl), _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags),
                                 _ptr(workspace),
                                 0 if workspace is None else workspace.numel(), _stream(stream)),
           "casc_syrk_fp64x2")
    return C_hi, C_lo, flags


_sig("casc_i8_gemm_fp64x2_ex", [ctypes.c_int, ctypes.c_int, _i64, _i64, _i64, ctypes.c_double,
                                ctypes.c_double, _vp, _vp, _i64, _vp, _vp, _i64, ctypes.c_double,
                                ctypes.c_double, _vp, _vp, _i64, _vp, ctypes.c_int, _vp, _sz,
                                _vp])


def casc_gemm_fp64x2_ex(transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo,
                        flags=None, workspace=None, stream=None):
    """C := alpha op(A) op(B) + beta C (FP64x2; NEXT-4).  transa/transb in
    {'N', 'T', 0, 1}; alpha, beta are (hi, lo) pairs or floats.  C_hi / C_lo
    (m x n) are updated in place; returns (C_hi, C_lo, flags)."""
    return _gemm_ex(None, transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo,
                    flags, workspace, stream)


def casc_i8_gemm_fp64x2_ex(transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo,
                           flags=None, y: int = 14, workspace=None, stream=None):
    """casc_gemm_fp64x2_ex on the INT8 cascade (NEXT-3 + NEXT-4): the product
    op(A) op(B) through y int8 slices (readings R21-R26)."""
    return _gemm_ex(int(y), transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo,
                    flags, workspace, stream)


def _gemm_ex(y, transa, transb, alpha, A_hi, A_lo, B_hi, B_lo, beta, C_hi, C_lo, flags,
             workspace, stream):
    ta = 1 if transa in ("T", "t", 1, True) else 0
    tb = 1 if transb in ("T", "t", 1, True) else 0
    ah, al = (alpha, 0.0) if isinstance(alpha, (int, float)) else alpha
    bh, bl = (beta, 0.0) if isinstance(beta, (int, float)) else beta
    m, n = C_hi.shape
    ldc = _ld_pair(C_hi, C_lo, "C")
    no_product = A_hi is None
    if not no_product:
        lda = _ld_pair(A_hi, A_lo, "A")
        ldb = _ld_pair(B_hi, B_lo, "B")
        k = A_hi.shape[0] if ta else A_hi.shape[1]
    else:
        lda = ldb = 1
        k = 0
    if flags is not None and (flags.dtype != torch.uint8 or tuple(flags.shape) != (m, n)):
        raise TypeError("flags must be a contiguous (m, n) uint8 CUDA tensor")
    head = (ta, tb, m, n, k, float(ah), float(al), _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
            _ptr(B_lo), ldb, float(bh), float(bl), _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags))
    tail = (_ptr(workspace), 0 if workspace is None else workspace.numel(), _stream(stream))
    if y is None:
        _check(_lib.casc_gemm_fp64x2_ex(*head, *tail), "casc_gemm_fp64x2_ex")
    else:
        _check(_lib.casc_i8_gemm_fp64x2_ex(*head, y, *tail), "casc_i8_gemm_fp64x2_ex")
    return C_hi, C_lo, flags


class CascError(RuntimeError):
    def __init__(self, status: int, fn: str):
        super().__init__(f"{fn}: {_lib.casc_status_string(status).decode()}")
        self.status = status


def _check(status: int, fn: str):
    if status != 0:
        raise CascError(status, fn)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def _mat(t, name):
    if t.dtype != torch.float64 or not t.is_cuda or t.dim() != 2:
        raise TypeError(f"{name} must be a 2-D float64 CUDA tensor")
    if t.size(1) > 1 and t.stride(1) != 1:
        raise TypeError(f"{name} must be row-major (unit column stride)")
    return max(t.stride(0), 1) if t.size(0) > 1 else max(t.size(1), 1)


def _hmat(t, name):
    if t.dtype != torch.float64 or t.is_cuda or t.dim() != 2:
        raise TypeError(f"{name} must be a 2-D float64 CPU (host) tensor")
    if t.size(1) > 1 and t.stride(1) != 1:
        raise TypeError(f"{name} must be row-major (unit column stride)")
    return max(t.stride(0), 1) if t.size(0) > 1 else max(t.size(1), 1)


def _ld_pair(hi, lo, name, host=False):
    ldh = (_hmat if host else _mat)(hi, name + "_hi")
    ldl = (_hmat if host else _mat)(lo, name + "_lo")
    if hi.shape != lo.shape or ldh != ldl:
        raise TypeError(f"{name}_hi and {name}_lo must have the same shape and layout")
    return ldh


def casc_status_string(status: int) -> str:
    return _lib.casc_status_string(status).decode()


def casc_select_widths(k: int):
    c = (ctypes.c_int * 3)()
    _check(_lib.casc_select_widths(k, c), "casc_select_widths")
    return tuple(c)


def casc_last_launch_count() -> int:
    return _lib.casc_last_launch_count()


def casc_workspace_bytes(m: int, n: int, k: int) -> int:
    return _lib.casc_workspace_bytes(m, n, k)


def casc_finalize():
    _check(_lib.casc_finalize(), "casc_finalize")


def _outputs(m, n, device, C_hi, C_lo, flags, want_flags, strided_flags=False):
    if C_hi is None:
        C_hi = torch.empty((m, n), dtype=torch.float64, device=device)
    if C_lo is None:
        C_lo = torch.empty((m, n), dtype=torch.float64, device=device)
    if flags is None and want_flags:
        flags = torch.empty((m, n), dtype=torch.uint8, device=device)
    if flags is not None:
        ok = flags.dtype == torch.uint8 and tuple(flags.shape) == (m, n)
        if strided_flags:
            ok = ok and (m * n == 0 or flags.stride(1) == 1)
        else:
            ok = ok and flags.is_contiguous()
        if not ok:
            raise TypeError("flags must be a (m, n) uint8 CUDA tensor (row-contiguous)")
    return C_hi, C_lo, flags


def _ldf(flags, n):
    return max(n, 1) if flags is None or flags.dim() != 2 or flags.shape[0] <= 1 \
        else flags.stride(0)


_sig("casc_gemm_fp64x2_host", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64,
                               _vp, _i64, _i64, _vp])


_sig("casc_i8_gemm_fp64x2_host", [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _vp, _vp,
                                  _i64, _vp, ctypes.c_int, _i64, _i64, _vp])


def casc_gemm_fp64x2_host(A_hi, A_lo, B_hi, B_lo, C_hi=None, C_lo=None, flags=None,
                          want_flags=True, slab_rows: int = 0, slab_cols: int = 0, stream=None,
                          sync: bool = True):
    """C := A B with HOST (CPU) tensors, streamed through the GPU in row slabs
    (casc.h: casc_gemm_fp64x2_host; bitwise the device-resident result).
    Pinned tensors (`.pin_memory()`) let the copies overlap the kernels.
    Outputs are pinned CPU tensors unless given.  sync=False returns right after
    enqueueing (the tensors must stay alive until `stream` completes)."""
    return _host_call(None, A_hi, A_lo, B_hi, B_lo, C_hi, C_lo, flags, want_flags, slab_rows,
                      slab_cols, stream, sync)


def casc_i8_gemm_fp64x2_host(A_hi, A_lo, B_hi, B_lo, y: int = 14, C_hi=None, C_lo=None,
                             flags=None, want_flags=True, slab_rows: int = 0, slab_cols: int = 0,
                             stream=None, sync: bool = True):
    """casc_gemm_fp64x2_host on the INT8 cascade (NEXT-3; casc_i8_gemm_fp64x2_host)."""
    return _host_call(int(y), A_hi, A_lo, B_hi, B_lo, C_hi, C_lo, flags, want_flags, slab_rows,
                      slab_cols, stream, sync)


def _host_call(y, A_hi, A_lo, B_hi, B_lo, C_hi, C_lo, flags, want_flags, slab_rows, slab_cols,
               stream, sync):
    lda = _ld_pair(A_hi, A_lo, "A", host=True)
    ldb = _ld_pair(B_hi, B_lo, "B", host=True)
    m, k = A_hi.shape
    k2, n = B_hi.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    pin = lambda t: t.pin_memory() if torch.cuda.is_available() else t
    if C_hi is None:
        C_hi = pin(torch.empty((m, n), dtype=torch.float64))
    if C_lo is None:
        C_lo = pin(torch.empty((m, n), dtype=torch.float64))
    if flags is None and want_flags:
        flags = pin(torch.empty((m, n), dtype=torch.uint8))
    if flags is not None and (flags.dtype != torch.uint8 or flags.is_cuda
                              or not flags.is_contiguous() or tuple(flags.shape) != (m, n)):
        raise TypeError("flags must be a contiguous (m, n) uint8 CPU tensor")
    ldc = _ld_pair(C_hi, C_lo, "C", host=True)
    head = (m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi), _ptr(B_lo), ldb, _ptr(C_hi),
            _ptr(C_lo), ldc, _ptr(flags))
    if y is None:
        _check(_lib.casc_gemm_fp64x2_host(*head, int(slab_rows), int(slab_cols),
                                          _stream(stream)), "casc_gemm_fp64x2_host")
    else:
        _check(_lib.casc_i8_gemm_fp64x2_host(*head, y, int(slab_rows), int(slab_cols),
                                             _stream(stream)),
               "casc_i8_gemm_fp64x2_host")
    if sync:
        (stream or torch.cuda.current_stream()).synchronize()
    return C_hi, C_lo, flags


def casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=None, C_lo=None, flags=None,
                     want_flags=True, stream=None, workspace=None):
    """C := A B (cascaded FP64x2).  Returns (C_hi, C_lo, flags).  With
    `workspace` (uint8 CUDA tensor of casc_workspace_bytes(m, n, k)) this calls
    casc_gemm_fp64x2_ws, otherwise a stream-ordered per-call workspace is used."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    k2, n = B_hi.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    C_hi, C_lo, flags = _outputs(m, n, A_hi.device, C_hi, C_lo, flags, want_flags)
    ldc = _ld_pair(C_hi, C_lo, "C")
    if workspace is None:
        st = _lib.casc_gemm_fp64x2(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi), _ptr(B_lo),
                                   ldb, _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags), _stream(stream))
        _check(st, "casc_gemm_fp64x2")
    else:
        st = _lib.casc_gemm_fp64x2_ws(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                      _ptr(B_lo), ldb, _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags),
                                      _ptr(workspace), workspace.numel(), _stream(stream))
        _check(st, "casc_gemm_fp64x2_ws")
    return C_hi, C_lo, flags


def casc_gemm_fp64x2_ws(A_hi, A_lo, B_hi, B_lo, workspace, **kw):
    return casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, workspace=workspace, **kw)


def casc_packed_a_bytes(m: int, k: int) -> int:
    return _lib.casc_packed_a_bytes(m, k)


def casc_packed_b_bytes(k: int, n: int) -> int:
    return _lib.casc_packed_b_bytes(k, n)


def casc_packed_a_block_bytes(k: int) -> int:
    return _lib.casc_packed_a_block_bytes(k)


def casc_packed_b_block_bytes(k: int) -> int:
    return _lib.casc_packed_b_block_bytes(k)


def casc_pack_a(A_hi, A_lo, packed=None, stream=None):
    """Phase 1 for A into the opaque packed layout (uint8 CUDA tensor)."""
    lda = _ld_pair(A_hi, A_lo, "A")
    m, k = A_hi.shape
    if packed is None:
        packed = torch.empty(casc_packed_a_bytes(m, k), dtype=torch.uint8, device=A_hi.device)
    _check(_lib.casc_pack_a(m, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(packed), _stream(stream)),
           "casc_pack_a")
    return packed


def casc_pack_b(B_hi, B_lo, packed=None, stream=None):
    """Phase 1 for B (7 slices) into the opaque packed layout."""
    ldb = _ld_pair(B_hi, B_lo, "B")
    k, n = B_hi.shape
    if packed is None:
        packed = torch.empty(casc_packed_b_bytes(k, n), dtype=torch.uint8, device=B_hi.device)
    _check(_lib.casc_pack_b(k, n, _ptr(B_hi), _ptr(B_lo), ldb, _ptr(packed), _stream(stream)),
           "casc_pack_b")
    return packed


def casc_gemm_packed(m, n, k, packed_a, packed_b, C_hi=None, C_lo=None, flags=None,
                     want_flags=True, stream=None):
    """Phases 2-3 from packed operands.  Returns (C_hi, C_lo, flags).  C and
    flags may be column blocks of larger row-major arrays (casc_gemm_packed_ld)."""
    dev = packed_a.device if packed_a is not None else torch.device("cuda")
    C_hi, C_lo, flags = _outputs(m, n, dev, C_hi, C_lo, flags, want_flags, strided_flags=True)
    ldc = _ld_pair(C_hi, C_lo, "C") if m and n else max(n, 1)
    _check(_lib.casc_gemm_packed_ld(m, n, k, _ptr(packed_a), _ptr(packed_b), _ptr(C_hi),
                                    _ptr(C_lo), ldc, _ptr(flags), _ldf(flags, n),
                                    _stream(stream)), "casc_gemm_packed_ld")
    return C_hi, C_lo, flags


def casc_split_a(A_hi, A_lo, stream=None):
    """Slices (4, m, k) in the paper's normalisation and exponents (P, m)."""
    lda = _ld_pair(A_hi, A_lo, "A")
    m, k = A_hi.shape
    P = (k + KC - 1) // KC
    S = torch.empty((4, m, k), dtype=torch.float64, device=A_hi.device)
    e = torch.empty((P, m), dtype=torch.int32, device=A_hi.device)
    _check(_lib.casc_split_a(m, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(S), _ptr(e),
                             _stream(stream)), "casc_split_a")
    return S, e


def casc_split_b(B_hi, B_lo, stream=None):
    """Slices (7, k, n) = B0..B6 in the paper's normalisation and exponents (P, n)."""
    ldb = _ld_pair(B_hi, B_lo, "B")
    k, n = B_hi.shape
    P = (k + KC - 1) // KC
    S = torch.empty((7, k, n), dtype=torch.float64, device=B_hi.device)
    f = torch.empty((P, n), dtype=torch.int32, device=B_hi.device)
    _check(_lib.casc_split_b(k, n, _ptr(B_hi), _ptr(B_lo), ldb, _ptr(S), _ptr(f),
                             _stream(stream)), "casc_split_b")
    return S, f


def casc_debug_bins(A_hi, A_lo, B_hi, B_lo, panel: int, stream=None):
    """Bins (4, m, n) of k panel `panel` as computed by the fused kernel."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    n = B_hi.shape[1]
    bins = torch.empty((4, m, n), dtype=torch.float64, device=A_hi.device)
    _check(_lib.casc_debug_bins(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi), _ptr(B_lo),
                                ldb, panel, _ptr(bins), _stream(stream)), "casc_debug_bins")
    return bins


def casc_debug_ldexp(x, n, stream=None):
    """x * 2^n per element as the kernels scale (bitwise ldexp), x float64 and n
    int32 CUDA tensors of the same shape."""
    x = x.contiguous()
    n = n.to(torch.int32).contiguous()
    if x.shape != n.shape:
        raise ValueError("x and n differ in shape")
    out = torch.empty_like(x)
    _check(_lib.casc_debug_ldexp(x.numel(), _ptr(x), _ptr(n), _ptr(out), _stream(stream)),
           "casc_debug_ldexp")
    return out


def casc_gemm_fp64x2_simple(A_hi, A_lo, B_hi, B_lo, C_hi=None, C_lo=None, flags=None,
                            want_flags=True, stream=None):
    """The paper's simple path (§4.2): ten slice-GEMM launches into four HBM bins
    per panel + standalone epilogue.  Returns (C_hi, C_lo, flags)."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    k2, n = B_hi.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    C_hi, C_lo, flags = _outputs(m, n, A_hi.device, C_hi, C_lo, flags, want_flags)
    ldc = _ld_pair(C_hi, C_lo, "C")
    _check(_lib.casc_gemm_fp64x2_simple(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                        _ptr(B_lo), ldb, _ptr(C_hi), _ptr(C_lo), ldc,
                                        _ptr(flags), _stream(stream)),
           "casc_gemm_fp64x2_simple")
    return C_hi, C_lo, flags


def casc_slice_product(A_hi, A_lo, B_hi, B_lo, sa: int, sb: int, panel: int, stream=None):
    """One slice GEMM A_sa . B_sb of k panel `panel` (paper normalisation), (m, n)."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    n = B_hi.shape[1]
    out = torch.empty((m, n), dtype=torch.float64, device=A_hi.device)
    _check(_lib.casc_slice_product(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                   _ptr(B_lo), ldb, sa, sb, panel, _ptr(out), _stream(stream)),
           "casc_slice_product")
    return out


# ---------------------------------------------------------------- NEXT-3: INT8 cascade
def casc_i8_workspace_bytes(m: int, n: int, k: int, y: int = I8_DEFAULT_SLICES) -> int:
    return _lib.casc_i8_workspace_bytes(m, n, k, y)


def casc_i8_packed_bytes(rows: int, k: int, y: int = I8_DEFAULT_SLICES) -> int:
    return _lib.casc_i8_packed_bytes(rows, k, y)


def casc_i8_finalize():
    _check(_lib.casc_i8_finalize(), "casc_i8_finalize")


def casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, y: int = I8_DEFAULT_SLICES, C_hi=None,
                        C_lo=None, flags=None, want_flags=True, stream=None, workspace=None):
    """C := A B through y int8 slices on the INT8 tensor cores (NEXT-3; readings
    R22-R26).  Returns (C_hi, C_lo, flags).  With `workspace` (uint8 CUDA tensor
    of casc_i8_workspace_bytes(m, n, k, y)) this calls casc_i8_gemm_fp64x2_ws."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    k2, n = B_hi.shape
    if k != k2:
        raise ValueError("inner dimensions differ")
    C_hi, C_lo, flags = _outputs(m, n, A_hi.device, C_hi, C_lo, flags, want_flags)
    ldc = _ld_pair(C_hi, C_lo, "C")
    if workspace is None:
        st = _lib.casc_i8_gemm_fp64x2(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                      _ptr(B_lo), ldb, _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags),
                                      int(y), _stream(stream))
        _check(st, "casc_i8_gemm_fp64x2")
    else:
        st = _lib.casc_i8_gemm_fp64x2_ws(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi),
                                         _ptr(B_lo), ldb, _ptr(C_hi), _ptr(C_lo), ldc,
                                         _ptr(flags), int(y), _ptr(workspace), workspace.numel(),
                                         _stream(stream))
        _check(st, "casc_i8_gemm_fp64x2_ws")
    return C_hi, C_lo, flags


def casc_i8_gemm_fp64x2_ws(A_hi, A_lo, B_hi, B_lo, workspace, **kw):
    return casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, workspace=workspace, **kw)


def casc_i8_split(hi, lo, is_b: bool, y: int = I8_DEFAULT_SLICES, stream=None):
    """Digits (y, rows, k) int8 and exponents (P, rows) int32 of A (is_b False,
    rows x k) or of B's columns (is_b True, B is k x rows), from the GEMM's own
    split kernels (R22, R23)."""
    ld = _ld_pair(hi, lo, "X")
    if is_b:
        k, rows = hi.shape
    else:
        rows, k = hi.shape
    P = (k + I8_KC - 1) // I8_KC
    D = torch.empty((y, rows, k), dtype=torch.int8, device=hi.device)
    E = torch.empty((P, rows), dtype=torch.int32, device=hi.device)
    _check(_lib.casc_i8_split(rows, k, _ptr(hi), _ptr(lo), ld, int(bool(is_b)), int(y), _ptr(D),
                              _ptr(E), _stream(stream)), "casc_i8_split")
    return D, E


def casc_i8_debug_bins(A_hi, A_lo, B_hi, B_lo, panel: int = 0, y: int = I8_DEFAULT_SLICES,
                       stream=None):
    """Exact int32 bins (y, m, n) of k panel `panel` as accumulated in tensor memory (R24)."""
    lda = _ld_pair(A_hi, A_lo, "A")
    ldb = _ld_pair(B_hi, B_lo, "B")
    m, k = A_hi.shape
    n = B_hi.shape[1]
    bins = torch.empty((y, m, n), dtype=torch.int32, device=A_hi.device)
    _check(_lib.casc_i8_debug_bins(m, n, k, _ptr(A_hi), _ptr(A_lo), lda, _ptr(B_hi), _ptr(B_lo),
                                   ldb, int(y), panel, _ptr(bins), _stream(stream)),
           "casc_i8_debug_bins")
    return bins


def casc_i8_packed_block_bytes(k: int, y: int = I8_DEFAULT_SLICES) -> int:
    return _lib.casc_i8_packed_block_bytes(k, y)


def casc_i8_gemm_ws_bytes(m: int, n: int) -> int:
    return _lib.casc_i8_gemm_ws_bytes(m, n)


def casc_i8_pack(hi, lo, is_b: bool, y: int = I8_DEFAULT_SLICES, packed=None, stream=None):
    """Phase 1 of the INT8 cascade into the opaque packed layout (uint8 CUDA tensor):
    A (rows x k) or, with is_b, B (k x rows, packed per column)."""
    ld = _ld_pair(hi, lo, "X")
    k, rows = hi.shape if is_b else hi.shape[::-1]
    if packed is None:
        packed = torch.empty(casc_i8_packed_bytes(rows, k, y), dtype=torch.uint8,
                             device=hi.device)
    _check(_lib.casc_i8_pack(rows, k, _ptr(hi), _ptr(lo), ld, int(bool(is_b)), int(y),
                             _ptr(packed), _stream(stream)), "casc_i8_pack")
    return packed


def casc_i8_gemm_packed(m, n, k, packed_a, packed_b, y: int = I8_DEFAULT_SLICES, C_hi=None,
                        C_lo=None, flags=None, want_flags=True, ws=None, stream=None):
    """Phases 2-3 of the INT8 cascade from packed operands.  Returns (C_hi, C_lo, flags).
    C and flags may be column blocks of larger arrays (casc_i8_gemm_packed_ld)."""
    dev = packed_a.device if packed_a is not None else torch.device("cuda")
    C_hi, C_lo, flags = _outputs(m, n, dev, C_hi, C_lo, flags, want_flags, strided_flags=True)
    ldc = _ld_pair(C_hi, C_lo, "C") if m and n else max(n, 1)
    if ws is None:
        ws = torch.empty(max(casc_i8_gemm_ws_bytes(m, n), 1), dtype=torch.uint8, device=dev)
    _check(_lib.casc_i8_gemm_packed_ld(m, n, k, int(y), _ptr(packed_a), _ptr(packed_b),
                                       _ptr(C_hi), _ptr(C_lo), ldc, _ptr(flags), _ldf(flags, n),
                                       _ptr(ws), ws.numel(), _stream(stream)),
           "casc_i8_gemm_packed_ld")
    return C_hi, C_lo, flags


# ------------------------------------------------------------ peer-memory exchange
# (include/casc.h: casc_ipc_alloc / _free / _open / _close, casc_copy_async)
_sig("casc_ipc_alloc", [_sz, ctypes.POINTER(_vp), _vp])
_sig("casc_ipc_free", [_vp])
_sig("casc_ipc_open", [_vp, ctypes.POINTER(_vp)])
_sig("casc_ipc_close", [_vp])
_sig("casc_copy_async", [_vp, _vp, _sz, _vp])
CASC_IPC_HANDLE_BYTES = 64
EXPORTED += ["casc_ipc_alloc", "casc_ipc_free", "casc_ipc_open", "casc_ipc_close",
             "casc_copy_async"]


class _DevBuf:
    """__cuda_array_interface__ of a raw device byte range (for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1",
                                         "data": (ptr, False), "version": 3, "strides": None}


def casc_ipc_alloc(nbytes: int):
    """Exported device buffer: (ptr, handle bytes, uint8 tensor view of it)."""
    ptr = _vp()
    handle = ctypes.create_string_buffer(CASC_IPC_HANDLE_BYTES)
    _check(_lib.casc_ipc_alloc(int(nbytes), ctypes.byref(ptr), handle), "casc_ipc_alloc")
    view = torch.as_tensor(_DevBuf(ptr.value, int(nbytes)), device="cuda")
    return ptr.value, handle.raw, view


def casc_ipc_free(ptr: int):
    _check(_lib.casc_ipc_free(ptr), "casc_ipc_free")


def casc_ipc_open(handle: bytes) -> int:
    """Map another process's exported buffer; returns its base address here."""
    if len(handle) != CASC_IPC_HANDLE_BYTES:
        raise ValueError("IPC handle must be 64 bytes")
    ptr = _vp()
    buf = ctypes.create_string_buffer(handle, CASC_IPC_HANDLE_BYTES)
    _check(_lib.casc_ipc_open(buf, ctypes.byref(ptr)), "casc_ipc_open")
    return ptr.value


def casc_ipc_close(ptr: int):
    _check(_lib.casc_ipc_close(ptr), "casc_ipc_close")


def casc_copy_async(dst: int, src: int, nbytes: int, stream=None):
    """Enqueue a copy-engine copy (cudaMemcpyDefault) of nbytes on `stream`."""
    _check(_lib.casc_copy_async(dst, src, int(nbytes), _stream(stream)), "casc_copy_async")
