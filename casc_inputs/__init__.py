"""Seeded synthetic FP64x2 inputs shared by the oracle tests, the GPU parity
tests and bench.py.

This module holds NONE of the method's arithmetic (no split, no bins, no
double-double operations): it only draws counter-based random numbers and
places them, so that both sides of every parity test see identical inputs.

Recipe (stand-ins for the paper's generators, and
BASELINE.json configs 0-4):

* RNG: counter-based splitmix64.  For (seed, stream, index) the 64-bit state is
  ``x = seed*0x9E3779B97F4A7C15 + stream*0xD1B54A32D192ED03 + (index+1)*0xBF58476D1CE4E5B9``
  (mod 2^64), finalised by the splitmix64 mixer.  ``u = (z >> 11) * 2^-53``
  lies in [0, 1); ``U = 2u - 1`` lies in [-1, 1) on the 2^-52 grid.
  The index is the global row-major element index, so any row block or column
  slab of a matrix is bit-identical to the same block of the full matrix (this
  is what makes the multi-GPU P-invariance test meaningful).
* FP64x2 element: ``h = U``, ``l = RN(RN(h * 2^-53) * U')`` with U' from
  another stream (BASELINE: "lo = hi*2^-53*Uniform[-1,1]"); |l| can reach
  ulp(h), so the pair is renormalised once with Dekker's Fast2Sum
  (``hi = RN(h + l)``, ``lo = l - (hi - h)``, exact since |h| >= |l|) to meet
  the non-overlap precondition |lo| <= ulp(hi)/2 (DESIGN.md reading
  R15).  This is input preparation, not the method's arithmetic.
* Streams: 0 A.hi, 1 A.lo factor, 2 B.hi, 3 B.lo factor, 4 row exponents u,
  5 column exponents v, 6 perturbation, 7 pairing perturbation.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_G = np.uint64(0x9E3779B97F4A7C15)
_S = np.uint64(0xD1B54A32D192ED03)
_I = np.uint64(0xBF58476D1CE4E5B9)
_C1 = np.uint64(0xBF58476D1CE4E5B9)
_C2 = np.uint64(0x94D049BB133111EB)

STREAM_A_HI, STREAM_A_LO, STREAM_B_HI, STREAM_B_LO = 0, 1, 2, 3
STREAM_ROW_EXP, STREAM_COL_EXP, STREAM_PERTURB, STREAM_PAIR = 4, 5, 6, 7


def splitmix64(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """splitmix64 finaliser of the counter state for uint64 indices."""
    with np.errstate(over="ignore"):
        idx = np.asarray(index, dtype=np.uint64)
        x = (np.uint64(seed & 0xFFFFFFFFFFFFFFFF) * _G
             + np.uint64(stream) * _S
             + (idx + np.uint64(1)) * _I)
        z = x
        z = (z ^ (z >> np.uint64(30))) * _C1
        z = (z ^ (z >> np.uint64(27))) * _C2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """u in [0, 1) on the 2^-53 grid."""
    z = splitmix64(seed, stream, index)
    return (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_pm1(seed: int, stream: int, index: np.ndarray) -> np.ndarray:
    """U in [-1, 1) on the 2^-52 grid (exact: 2u - 1 with u on the 2^-53 grid)."""
    return 2.0 * uniform01(seed, stream, index) - 1.0


def _renormalise(h: np.ndarray, l: np.ndarray):
    """Dekker Fast2Sum (|h| >= |l|): the exact normalised pair for h + l."""
    s = h + l
    return s, l - (s - h)


def _grid_index(rows: slice, cols: slice, ncols: int) -> np.ndarray:
    r = np.arange(rows.start, rows.stop, dtype=np.uint64)[:, None]
    c = np.arange(cols.start, cols.stop, dtype=np.uint64)[None, :]
    return r * np.uint64(ncols) + c


def dd_uniform(seed: int, hi_stream: int, lo_stream: int, nrows: int, ncols: int,
               rows: slice | None = None, cols: slice | None = None,
               chunk_rows: int = 512):
    """(hi, lo) arrays of the uniform FP64x2 distribution (BASELINE configs 0, 1, 4):
    hi ~ U[-1,1) and lo = hi * 2^-53 * U'.  Optionally only a sub-block."""
    rows = rows or slice(0, nrows)
    cols = cols or slice(0, ncols)
    m = rows.stop - rows.start
    n = cols.stop - cols.start
    hi = np.empty((m, n), dtype=np.float64)
    lo = np.empty((m, n), dtype=np.float64)
    chunk_rows = max(1, min(chunk_rows, (1 << 22) // max(n, 1)))

    def fill(r0):
        r1 = min(m, r0 + chunk_rows)
        idx = _grid_index(slice(rows.start + r0, rows.start + r1), cols, ncols)
        h = uniform_pm1(seed, hi_stream, idx)
        l = (h * (2.0 ** -53)) * uniform_pm1(seed, lo_stream, idx)
        hi[r0:r1], lo[r0:r1] = _renormalise(h, l)

    starts = list(range(0, m, chunk_rows))
    if len(starts) > 1:
        # numpy ufuncs release the GIL: chunks fill in parallel, output unchanged
        with ThreadPoolExecutor(max_workers=min(32, os.cpu_count() or 1)) as ex:
            list(ex.map(fill, starts))
    else:
        for r0 in starts:
            fill(r0)
    return hi, lo


def int_uniform(seed: int, stream: int, count: int, lo: int, hi: int) -> np.ndarray:
    """Integers uniform in [lo, hi] (inclusive) from stream `stream`."""
    u = uniform01(seed, stream, np.arange(count, dtype=np.uint64))
    return (lo + np.floor(u * (hi - lo + 1))).astype(np.int64)


def make_config(cfg: int, seed: int | None = None, m: int | None = None,
                n: int | None = None, k: int | None = None, variant: str = "a",
                rows: slice | None = None, cols: slice | None = None):
    """Inputs for BASELINE.json config `cfg` (optionally shrunk to m, n, k for
    parity tests that keep the structure but not the size).

    Returns dict(A_hi, A_lo, B_hi, B_lo, m, n, k, name).

    cfg 0: 64^3 uniform, seed 0.          cfg 1: 1024^3 uniform.
    cfg 2: 4096^3, row i of A scaled by 2^u_i, column j of B by 2^v_j,
           u, v ~ U_int[-30, 30].
    cfg 3: m=n=4096, k=32768 engineered cancellation (reading R13):
           variant "a": literal - B[:, n/2 + j] = -B[:, j] + 2^-60 U (the
                        perturbation enters the lo limb);
           variant "b": in-panel pairing - inside each 256-wide k panel,
                        A[:, p+128] = A[:, p], B[p+128, :] = -B[p, :] + 2^-60 U;
           variant "c": cross-panel pairing - A[:, p+256] = A[:, p],
                        B[p+256, :] = -B[p, :] + 2^-60 U for even panels.
    cfg 4: 16384^3 uniform (headline; C row-block sharded over GPUs).
    `rows` restricts A (and the output) to a row block, `cols` restricts B (and
    the output) to a column slab; either block is bit-identical to the same
    block of the full matrices (global-index RNG).  (cfg 3 builds the full B and
    slices it: its column pairing crosses slabs.)
    """
    defaults = {0: (64, 64, 64), 1: (1024, 1024, 1024), 2: (4096, 4096, 4096),
                3: (4096, 4096, 32768), 4: (16384, 16384, 16384)}
    if cfg not in defaults:
        raise ValueError(f"unknown config {cfg}")
    dm, dn, dk = defaults[cfg]
    m = dm if m is None else m
    n = dn if n is None else n
    k = dk if k is None else k
    seed = cfg if seed is None else seed
    rows = rows or slice(0, m)
    cols = cols or slice(0, n)
    A_hi, A_lo = dd_uniform(seed, STREAM_A_HI, STREAM_A_LO, m, k, rows=rows)
    B_hi, B_lo = dd_uniform(seed, STREAM_B_HI, STREAM_B_LO, k, n,
                            cols=None if cfg == 3 else cols)
    name = f"cfg{cfg}_{m}x{n}x{k}"
    if cfg == 2:
        u = int_uniform(seed, STREAM_ROW_EXP, m, -30, 30)[rows]
        v = int_uniform(seed, STREAM_COL_EXP, n, -30, 30)[cols]
        su = np.ldexp(1.0, u)[:, None]
        sv = np.ldexp(1.0, v)[None, :]
        A_hi *= su
        A_lo *= su
        B_hi *= sv
        B_lo *= sv
    elif cfg == 3:
        name += variant
        if variant == "a":
            h = n // 2
            pert = uniform_pm1(seed, STREAM_PERTURB,
                               _grid_index(slice(0, k), slice(0, h), h)) * (2.0 ** -60)
            B_hi[:, h:2 * h] = -B_hi[:, :h]
            B_lo[:, h:2 * h] = -B_lo[:, :h] + pert
        elif variant in ("b", "c"):
            span = 128 if variant == "b" else 256
            period = 2 * span
            for p0 in range(0, k - span, period):
                w = min(span, k - span - p0)
                A_hi[:, p0 + span:p0 + span + w] = A_hi[:, p0:p0 + w]
                A_lo[:, p0 + span:p0 + span + w] = A_lo[:, p0:p0 + w]
                pert = uniform_pm1(seed, STREAM_PAIR,
                                   _grid_index(slice(p0, p0 + w), slice(0, n), n)) * (2.0 ** -60)
                B_hi[p0 + span:p0 + span + w, :] = -B_hi[p0:p0 + w, :]
                B_lo[p0 + span:p0 + span + w, :] = -B_lo[p0:p0 + w, :] + pert
        else:
            raise ValueError(f"unknown cfg3 variant {variant}")
        # the 2^-60 perturbation went into the lo limb: renormalise the pairs
        # (|lo| <= ulp(hi)/2 again for small |hi|; reading R15)
        B_hi, B_lo = _renormalise(B_hi, B_lo)
        B_hi = np.ascontiguousarray(B_hi[:, cols])
        B_lo = np.ascontiguousarray(B_lo[:, cols])
    return dict(A_hi=A_hi, A_lo=A_lo, B_hi=B_hi, B_lo=B_lo, m=m, n=n, k=k, name=name)


def full_mantissa(seed: int, nrows: int, ncols: int, max_shift: int = 40):
    """Full-mantissa distribution for split parity:
    hi = +-(1 + u) 2^-L with L ~ U_int[0, max_shift] per element, lo = hi 2^-53 U'.
    Exercises leading zeros and slice-3 rounding that U[-1,1] hides."""
    idx = _grid_index(slice(0, nrows), slice(0, ncols), ncols)
    u = uniform01(seed, STREAM_A_HI, idx)
    s = uniform01(seed, STREAM_PERTURB, idx)
    L = np.floor(uniform01(seed, STREAM_PAIR, idx) * (max_shift + 1))
    hi = np.where(s < 0.5, -1.0, 1.0) * np.ldexp(1.0 + u, -L.astype(np.int64))
    lo = (hi * (2.0 ** -53)) * uniform_pm1(seed, STREAM_A_LO, idx)
    return _renormalise(hi, lo)
