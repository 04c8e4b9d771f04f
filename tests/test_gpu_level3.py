"""GPU parity of the level-3 routines added in round 2 (NEXT-4, P:L3838-3839;
readings R28, R29): SYMM, TRMM and the right-side TRSM through the C ABI,
against their oracles (oracle/casc_oracle.c) and against the cascaded GEMM
they are built on."""

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


def _nan_other(hi, lo, uplo, unit=False):
    other = np.triu(np.ones(hi.shape, bool), 1) if uplo == "L" else \
        np.tril(np.ones(hi.shape, bool), -1)
    hi, lo = np.where(other, np.nan, hi), np.where(other, np.nan, lo)
    if unit:
        np.fill_diagonal(hi, np.nan)
        np.fill_diagonal(lo, np.nan)
    return hi, lo


@pytest.mark.parametrize("side,uplo,m,n", [("L", "L", 300, 200), ("R", "U", 130, 520),
                                           ("L", "U", 64, 1), ("R", "L", 1, 77)])
def test_symm_bitwise_gemm_and_oracle(casc, orc, side, uplo, m, n):
    """SYMM reads only the `uplo` triangle (NaN elsewhere) and is bitwise the
    cascaded GEMM of the full symmetric matrix; within twice the north-star
    bound of the oracle's SYMM, flags equal; the beta update as the GEMM's."""
    import torch
    ka = m if side == "L" else n
    d = I.make_config(2, m=ka, n=ka, k=ka, seed=51)
    tri = np.tril(np.ones((ka, ka), bool)) if uplo == "L" else np.triu(np.ones((ka, ka), bool))
    S_hi = np.where(tri, d["A_hi"], d["A_hi"].T)
    S_lo = np.where(tri, d["A_lo"], d["A_lo"].T)
    A_hi, A_lo = _nan_other(d["A_hi"], d["A_lo"], uplo)
    b = I.make_config(1, m=m, n=n, k=n, seed=53)
    B_hi, B_lo = b["A_hi"], b["A_lo"]
    C0 = np.random.default_rng(5).uniform(-1, 1, (m, n))
    al, be = (0.75, 2.0 ** -60), (-1.25, 0.0)
    C_hi, C_lo = T(C0), T(np.zeros((m, n)))
    fl = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    casc.casc_symm_fp64x2(side, uplo, al, T(A_hi), T(A_lo), T(B_hi), T(B_lo), be, C_hi, C_lo,
                          flags=fl)
    G_hi, G_lo = T(C0), T(np.zeros((m, n)))
    gfl = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    ops = (T(S_hi), T(S_lo), T(B_hi), T(B_lo)) if side == "L" else \
        (T(B_hi), T(B_lo), T(S_hi), T(S_lo))
    casc.casc_gemm_fp64x2_ex("N", "N", al, *ops, be, G_hi, G_lo, flags=gfl)
    assert np.array_equal(bits(N(C_hi)), bits(N(G_hi))) and np.array_equal(bits(N(C_lo)), bits(N(G_lo)))
    assert np.array_equal(N(fl), N(gfl))
    o_hi, o_lo, o_fl = orc.casc_symm(side, uplo, al, A_hi, A_lo, B_hi, B_lo, be, C0,
                                     np.zeros((m, n)))
    assert np.array_equal(N(fl), o_fl)
    L = (S_hi, S_lo, B_hi, B_lo) if side == "L" else (B_hi, B_lo, S_hi, S_lo)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(*L, ii.ravel(), jj.ravel())
    bound = (abs(al[0]) * 2 * orc.north_star_bound(ka, r["absab"])).reshape(m, n) \
        + 2.0 ** -100 * np.abs(o_hi)
    assert np.all(np.abs((N(C_hi) - o_hi) + (N(C_lo) - o_lo)) <= bound)


@pytest.mark.parametrize("side,uplo,trans,diag,m,n", [("L", "L", "N", "N", 300, 90),
                                                      ("L", "U", "T", "U", 257, 33),
                                                      ("R", "L", "T", "N", 70, 600),
                                                      ("R", "U", "N", "U", 40, 129)])
def test_trmm_bitwise_gemm_and_oracle(casc, orc, side, uplo, trans, diag, m, n):
    """TRMM reads only A's triangle (NaN elsewhere / on a unit diagonal), is
    bitwise the cascaded GEMM of the triangular matrix, and is within twice the
    north-star bound of the oracle's TRMM; alpha = 0 zeroes B."""
    import torch
    ka = m if side == "L" else n
    d = I.make_config(1, m=ka, n=ka, k=ka, seed=57)
    tri = np.tril(np.ones((ka, ka), bool)) if uplo == "L" else np.triu(np.ones((ka, ka), bool))
    F_hi, F_lo = np.where(tri, d["A_hi"], 0.0), np.where(tri, d["A_lo"], 0.0)
    if diag == "U":
        np.fill_diagonal(F_hi, 1.0)
        np.fill_diagonal(F_lo, 0.0)
    A_hi, A_lo = _nan_other(d["A_hi"], d["A_lo"], uplo, diag == "U")
    b = I.make_config(1, m=m, n=n, k=n, seed=59)
    B_hi, B_lo = b["A_hi"], b["A_lo"]
    X_hi, X_lo = T(B_hi), T(B_lo)
    casc.casc_trmm_fp64x2(side, uplo, diag, 1.0, T(A_hi), T(A_lo), X_hi, X_lo, trans=trans)
    G_hi = torch.empty((m, n), dtype=torch.float64, device="cuda")
    G_lo = torch.empty_like(G_hi)
    if side == "L":
        casc.casc_gemm_fp64x2_ex(trans, "N", 1.0, T(F_hi), T(F_lo), T(B_hi), T(B_lo), 0.0, G_hi, G_lo)
    else:
        casc.casc_gemm_fp64x2_ex("N", trans, 1.0, T(B_hi), T(B_lo), T(F_hi), T(F_lo), 0.0, G_hi, G_lo)
    assert np.array_equal(bits(N(X_hi)), bits(N(G_hi))) and np.array_equal(bits(N(X_lo)), bits(N(G_lo)))
    o_hi, o_lo = orc.casc_trmm(side, uplo, diag, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    opF = (F_hi.T.copy(), F_lo.T.copy()) if trans == "T" else (F_hi, F_lo)
    L = (*opF, B_hi, B_lo) if side == "L" else (B_hi, B_lo, *opF)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(*L, ii.ravel(), jj.ravel())
    assert np.all(np.abs((N(X_hi) - o_hi) + (N(X_lo) - o_lo)).ravel()
                  <= 2 * orc.north_star_bound(ka, r["absab"]))
    Z_hi, Z_lo = T(B_hi), T(B_lo)
    casc.casc_trmm_fp64x2(side, uplo, diag, 0.0, T(np.full_like(A_hi, np.nan)),
                          T(np.full_like(A_lo, np.nan)), Z_hi, Z_lo, trans=trans)
    assert np.all(N(Z_hi) == 0) and np.all(N(Z_lo) == 0)


def _tri_dd(m, uplo, seed, unit=False):
    rng = np.random.default_rng(seed)
    hi = rng.uniform(-1, 1, (m, m)) / m
    hi = np.tril(hi) if uplo == "L" else np.triu(hi)
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, (m, m))
    d = 1.0 + rng.uniform(0, 1, m)
    hi[np.arange(m), np.arange(m)] = 1.0 if unit else d
    lo[np.arange(m), np.arange(m)] = 0.0 if unit else d * 2.0 ** -54
    s = hi + lo
    return s, lo - (s - hi)


@pytest.mark.parametrize("uplo,trans,diag,m,n", [("L", "N", "N", 70, 300), ("U", "N", "N", 33, 600),
                                                 ("L", "T", "U", 20, 1100), ("U", "T", "N", 9, 1300),
                                                 ("U", "N", "N", 1, 1), ("L", "N", "N", 5, 257)])
def test_trsm_right_vs_oracle_and_residual(casc, orc, uplo, trans, diag, m, n):
    """Right-side TRSM (column blocks, R29) against the oracle's (the left TRSM
    on the transposed system, R27: a different algorithm) to 2^-92 relative,
    the exact residual X op(A) - B within 2^-94 |X||op(A)| on sampled rows,
    alpha = 4 scales exactly, B as a column window of a wider buffer."""
    A_hi, A_lo = _tri_dd(n, uplo, 61, diag == "U")
    if diag == "U":
        A_hi = A_hi.copy()
        A_hi[np.arange(n), np.arange(n)] = np.nan  # the unit diagonal is not read
    rng = np.random.default_rng(63)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    Xh, Xl = T(B_hi), T(B_lo)
    casc.casc_trsm_fp64x2_right(uplo, diag, 1.0, T(A_hi), T(A_lo), Xh, Xl, trans=trans)
    x_hi, x_lo = N(Xh), N(Xl)
    o_hi, o_lo = orc.casc_trsm_right(uplo, diag, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    diff = np.abs((x_hi - o_hi) + (x_lo - o_lo))
    assert np.all(diff <= 2.0 ** -92 * (np.abs(o_hi) + 2.0 ** -20))
    A_use = A_hi.copy()
    if diag == "U":
        A_use[np.arange(n), np.arange(n)] = 1.0
    opA = (A_use.T.copy(), A_lo.T.copy()) if trans == "T" else (A_use, A_lo)
    rows = np.unique(np.linspace(0, m - 1, 4).astype(int))
    ii, jj = np.meshgrid(rows, np.arange(n), indexing="ij")
    r = orc.exact_entries(x_hi, x_lo, opA[0], opA[1], ii.ravel(), jj.ravel(), B_hi, B_lo)
    assert np.all(np.abs(r["err"]) <= 2.0 ** -94 * r["absab"] + 2.0 ** -120)
    wide_h = T(np.pad(B_hi, ((0, 0), (0, 3)), constant_values=5.0))
    wide_l = T(np.pad(B_lo, ((0, 0), (0, 3)), constant_values=5.0))
    casc.casc_trsm_fp64x2_right(uplo, diag, 4.0, T(A_hi), T(A_lo), wide_h[:, :n], wide_l[:, :n],
                                trans=trans)
    assert np.array_equal(N(wide_h)[:, :n], 4 * x_hi) and np.array_equal(N(wide_l)[:, :n], 4 * x_lo)
    assert np.all(N(wide_h)[:, n:] == 5.0)


def test_level3_bad_arguments(casc):
    import torch
    z = torch.zeros((4, 4), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        casc.casc_symm_fp64x2("X", "L", 1.0, z, z, z, z, 0.0, z.clone(), z.clone())
    with pytest.raises(ValueError):
        casc.casc_trmm_fp64x2("L", "Q", "N", 1.0, z, z, z.clone(), z.clone())
    with pytest.raises(casc.CascError):  # B overlapping A
        buf = torch.zeros((5, 4), dtype=torch.float64, device="cuda")
        casc.casc_trsm_fp64x2_right("L", "N", 1.0, buf[:4], buf[:4], buf[1:], buf[1:])


@pytest.mark.parametrize("uplo,trans,n,k", [("L", "N", 200, 300), ("U", "T", 130, 513),
                                            ("L", "T", 1100, 256)])
def test_syr2k_bitwise_gemms_and_oracle(casc, orc, uplo, trans, n, k):
    """SYR2K (R30): every stored element bitwise the two cascaded GEMM updates
    C := alpha op(A) op(B)^T + beta C; C := alpha op(B) op(A)^T + C of
    casc_gemm_fp64x2_ex (the triangular kernel computes the same tiles), the
    other triangle keeps its sentinel, flags = OR of the two GEMMs' flags and
    equal the oracle's; within twice the bound of the oracle."""
    import torch
    a = I.make_config(1, m=k, n=k, k=k, seed=91)
    b = I.make_config(2, m=k, n=k, k=k, seed=93)
    rows = min(n, k)
    A_hi = np.concatenate([a["A_hi"]] * (-(-n // k)))[:n]
    A_lo = np.concatenate([a["A_lo"]] * (-(-n // k)))[:n]
    B_hi = np.concatenate([b["A_hi"]] * (-(-n // k)))[:n]
    B_lo = np.concatenate([b["A_lo"]] * (-(-n // k)))[:n]
    A_hi[5], A_lo[5] = 0.0, 0.0
    B_hi[5], B_lo[5] = 0.0, 0.0
    st = (lambda x: x.T.copy()) if trans == "T" else (lambda x: x.copy())
    Ah, Al, Bh, Bl = (T(st(x)) for x in (A_hi, A_lo, B_hi, B_lo))
    C0 = np.random.default_rng(7).uniform(-1, 1, (n, n))
    al, be = (0.75, 2.0 ** -60), (-0.5, 0.0)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    C_hi = T(np.where(tri, C0, np.nan))
    C_lo = T(np.zeros((n, n)))
    fl = torch.full((n, n), 9, dtype=torch.uint8, device="cuda")
    casc.casc_syr2k_fp64x2(uplo, trans, al, Ah, Al, Bh, Bl, be, C_hi, C_lo, flags=fl)
    tb = "N" if trans == "T" else "T"
    G_hi, G_lo = T(C0), T(np.zeros((n, n)))
    f1 = torch.empty((n, n), dtype=torch.uint8, device="cuda")
    f2 = torch.empty((n, n), dtype=torch.uint8, device="cuda")
    casc.casc_gemm_fp64x2_ex(trans, tb, al, Ah, Al, Bh, Bl, be, G_hi, G_lo, flags=f1)
    casc.casc_gemm_fp64x2_ex(trans, tb, al, Bh, Bl, Ah, Al, 1.0, G_hi, G_lo, flags=f2)
    s_hi, s_lo, g_hi, g_lo = N(C_hi), N(C_lo), N(G_hi), N(G_lo)
    assert np.array_equal(bits(s_hi[tri]), bits(g_hi[tri])) and np.array_equal(bits(s_lo[tri]), bits(g_lo[tri]))
    assert np.all(np.isnan(s_hi[~tri]))
    f = N(fl)
    assert np.array_equal(f[tri], (N(f1) | N(f2))[tri]) and np.all(f[~tri] == 9)
    assert f[5][tri[5]].all()
    if n <= 200:
        o_hi, o_lo, o_fl = orc.casc_syr2k(uplo, trans, al, st(A_hi), st(A_lo), st(B_hi), st(B_lo),
                                          be, C0, np.zeros((n, n)))
        assert np.array_equal(f[tri], o_fl[tri])
        ii, jj = np.nonzero(tri)
        r1 = orc.exact_entries(A_hi, A_lo, B_hi.T.copy(), B_lo.T.copy(), ii, jj)
        r2 = orc.exact_entries(B_hi, B_lo, A_hi.T.copy(), A_lo.T.copy(), ii, jj)
        bound = 2 * abs(al[0]) * 2 * orc.north_star_bound(k, r1["absab"] + r2["absab"]) \
            + 2.0 ** -100 * np.abs(o_hi[tri])
        assert np.all(np.abs((s_hi[tri] - o_hi[tri]) + (s_lo[tri] - o_lo[tri])) <= bound)
