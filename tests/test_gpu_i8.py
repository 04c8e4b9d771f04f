"""GPU parity of the INT8 cascade (NEXT-3, readings R22-R26) through the C ABI
against the CPU oracle (oracle/casc_i8_oracle.c).

Every step of this variant is exact integer work or a fixed sequence of RNE
FP64 operations, so the bar is bit-exact everywhere:
  * int8 slices and scale exponents (R22, R23): bit-exact;
  * the int32 bins accumulated in tensor memory (R24): bit-exact;
  * C_hi, C_lo and the flags (R25, R26): bit-exact;
and, against ORACLE-EXACT, the north-star bound |C - C*| <= 4 k 2^-104 |A||B|.
Sizes span several 128 x 128 tiles with ragged edges, two k panels (k > 8192)
and the bench workload (sampled rows / columns: a row of C depends only on
that row of A and on B; a column only on that column of B and on A).
"""

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


def gpu_gemm(casc, d, y=14, **kw):
    return [N(x) for x in casc.casc_i8_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                                   T(d["B_lo"]), y=y, **kw)]


def bitwise(x, y):
    return np.array_equal(x.view(np.uint64), y.view(np.uint64))


SHAPES = [(0, 64, 64, 64), (1, 130, 257, 300), (2, 200, 129, 1000), (1, 1, 1, 1),
          (1, 3, 5, 9), (1, 128, 128, 128), (1, 40, 33, 8192 + 257)]


# ------------------------------------------------------------------ split (R22, R23)
@pytest.mark.parametrize("cfg,m,n,k", SHAPES)
def test_i8_split_bit_exact(casc, orc, cfg, m, n, k):
    d = I.make_config(cfg, m=m, n=n, k=k)
    DA, EA = (N(x) for x in casc.casc_i8_split(T(d["A_hi"]), T(d["A_lo"]), False))
    DB, EB = (N(x) for x in casc.casc_i8_split(T(d["B_hi"]), T(d["B_lo"]), True))
    for q, p0 in enumerate(range(0, k, 8192)):
        p1 = min(k, p0 + 8192)
        oa, oe = orc.i8_split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], 14)
        ob, of = orc.i8_split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], 14)
        assert np.array_equal(EA[q], oe) and np.array_equal(EB[q], of)
        assert np.array_equal(DA[:, :, p0:p1], oa)
        assert np.array_equal(DB[:, :, p0:p1], ob)


def test_i8_split_full_mantissa_and_slices(casc, orc):
    """Leading zeros, full mantissas and every slice count y = 3 .. 15."""
    hi, lo = I.full_mantissa(21, 70, 300, max_shift=60)
    for y in (3, 7, 14, 15):
        D, E = (N(x) for x in casc.casc_i8_split(T(hi), T(lo), False, y=y))
        od, oe = orc.i8_split_a_panel(hi, lo, y)
        assert np.array_equal(D, od) and np.array_equal(E[0], oe)


# ------------------------------------------------------------------ bins (R24)
@pytest.mark.parametrize("cfg,m,n,k,panel", [(1, 130, 257, 300, 0), (2, 64, 200, 1000, 0),
                                             (1, 40, 33, 8192 + 257, 1),
                                             (1, 40, 33, 8192 + 257, 0)])
def test_i8_bins_bit_exact(casc, orc, cfg, m, n, k, panel):
    d = I.make_config(cfg, m=m, n=n, k=k)
    bins = N(casc.casc_i8_debug_bins(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]),
                                     panel=panel))
    p0, p1 = panel * 8192, min(k, panel * 8192 + 8192)
    oa, _ = orc.i8_split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], 14)
    ob, _ = orc.i8_split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], 14)
    ob_bins = orc.i8_panel_bins(oa, ob)
    assert np.array_equal(bins.astype(np.int64), ob_bins)


# ------------------------------------------------------------------ C and flags (R25, R26)
@pytest.mark.parametrize("cfg,m,n,k", SHAPES)
def test_i8_gemm_bit_exact(casc, orc, cfg, m, n, k):
    d = I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo)
    assert np.array_equal(fl, ofl)


@pytest.mark.parametrize("y", [3, 5, 8, 15])
def test_i8_gemm_slice_counts(casc, orc, y):
    d = I.make_config(1, m=150, n=140, k=700, seed=y)
    C_hi, C_lo, fl = gpu_gemm(casc, d, y=y)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], y)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo) and np.array_equal(fl, ofl)


def test_i8_within_north_star_bound(casc, orc):
    d = I.make_config(2, m=160, n=150, k=2000, seed=5)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    ii, jj = np.meshgrid(np.arange(0, 160, 3), np.arange(0, 150, 7), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          C_hi, C_lo)
    assert np.max(np.abs(r["err"]) / orc.north_star_bound(2000, r["absab"])) <= 1.0
    assert fl.sum() == 0


@pytest.mark.parametrize("variant,expect", [("a", "none"), ("b", "all"), ("c", "all")])
def test_i8_cancellation_flags(casc, orc, variant, expect):
    """cfg3 structure (R13 with the 8192 panel of R22): flags identical to the
    oracle's; 3b / 3c cancel inside one panel and are flagged everywhere."""
    d = I.make_config(3, m=70, n=64, k=2048, variant=variant)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo) and np.array_equal(fl, ofl)
    assert (fl.sum() == 0) if expect == "none" else fl.all()


def test_i8_strided_and_edge_cases(casc, orc):
    import torch
    d = I.make_config(1, m=50, n=60, k=70, seed=3)
    # leading dimensions larger than the logical sizes (views into wider buffers)
    Ah = torch.zeros((50, 90), dtype=torch.float64, device="cuda")
    Al = torch.zeros_like(Ah)
    Bh = torch.zeros((70, 75), dtype=torch.float64, device="cuda")
    Bl = torch.zeros_like(Bh)
    Ah[:, :70] = T(d["A_hi"]); Al[:, :70] = T(d["A_lo"])
    Bh[:, :60] = T(d["B_hi"]); Bl[:, :60] = T(d["B_lo"])
    Ch = torch.full((50, 64), 7.0, dtype=torch.float64, device="cuda")
    Cl = torch.full((50, 64), 7.0, dtype=torch.float64, device="cuda")
    c_hi, c_lo, fl = casc.casc_i8_gemm_fp64x2(Ah[:, :70], Al[:, :70], Bh[:, :60], Bl[:, :60],
                                              C_hi=Ch[:, :60], C_lo=Cl[:, :60])
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert bitwise(N(c_hi), o_hi) and bitwise(N(c_lo), o_lo) and np.array_equal(N(fl), ofl)
    assert bool((Ch[:, 60:] == 7.0).all()) and bool((Cl[:, 60:] == 7.0).all())
    # k == 0: C := 0, flags := 0
    z = torch.zeros((4, 0), dtype=torch.float64, device="cuda")
    zb = torch.zeros((0, 3), dtype=torch.float64, device="cuda")
    c_hi, c_lo, fl = casc.casc_i8_gemm_fp64x2(z, z, zb, zb)
    assert not c_hi.any() and not c_lo.any() and not fl.any()
    # invalid slice counts
    with pytest.raises(casc.CascError):
        casc.casc_i8_gemm_fp64x2(Ah[:, :70], Al[:, :70], Bh[:, :60], Bl[:, :60], y=2)
    with pytest.raises(casc.CascError):
        casc.casc_i8_gemm_fp64x2(Ah[:, :70], Al[:, :70], Bh[:, :60], Bl[:, :60], y=16)


def test_i8_deterministic_and_workspace(casc, orc):
    import torch
    d = I.make_config(1, m=300, n=260, k=900, seed=8)
    a = gpu_gemm(casc, d)
    ws = torch.empty(casc.casc_i8_workspace_bytes(300, 260, 900), dtype=torch.uint8,
                     device="cuda")
    b = gpu_gemm(casc, d, workspace=ws)
    assert all(np.array_equal(x, z) for x, z in zip(a, b))


def test_i8_sampled_full_size_cfg1(casc, orc):
    """cfg1 (1024^3) in one launch, 24 sampled rows x all columns bit-exact."""
    d = I.make_config(1)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    rows = np.arange(0, 1024, 43)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"][rows], d["A_lo"][rows], d["B_hi"], d["B_lo"])
    assert bitwise(C_hi[rows], o_hi) and bitwise(C_lo[rows], o_lo)
    assert np.array_equal(fl[rows], ofl)


def test_i8_packed_interface_and_slab_contiguity(casc, orc):
    """casc_i8_pack + casc_i8_gemm_packed give the one-call result bit for bit,
    and a 256-column slab of B packs into exactly the matching byte range of the
    packed full B (the multi-GPU all-gather premise)."""
    import torch
    d = I.make_config(1, m=300, n=768, k=900, seed=12)
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    ref = [N(x) for x in casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)]
    pa = casc.casc_i8_pack(A_hi, A_lo, False)
    pb = casc.casc_i8_pack(B_hi, B_lo, True)
    got = [N(x) for x in casc.casc_i8_gemm_packed(300, 768, 900, pa, pb)]
    assert all(np.array_equal(x, z) for x, z in zip(ref, got))
    blk = casc.casc_i8_packed_block_bytes(900)
    assert pb.numel() == 6 * blk
    slab = casc.casc_i8_pack(B_hi[:, 256:512].contiguous(), B_lo[:, 256:512].contiguous(), True)
    assert slab.numel() == 2 * blk
    # chunks and exponents identical; the u64 max scratch is part of each block too
    assert torch.equal(slab, pb[2 * blk:4 * blk])


@pytest.mark.parametrize("cfg,variant", [(2, "a"), (3, "a"), (3, "b"), (4, "a")])
def test_i8_full_size_configs_sampled(casc, orc, cfg, variant):
    """BASELINE configs 2, 3 and 4 at FULL size through casc_i8_gemm_fp64x2 (the
    kernels and launch configuration bench.py times): a rows x 96-column block
    bit-exact against the INT8 oracle (rows and columns are independent: per-row
    and per-column scales), sampled entries within the north-star bound of the
    exact product (except where flagged: 3b cancels by design)."""
    import torch
    d = I.make_config(cfg, variant=variant)
    m, n, k = d["m"], d["n"], d["k"]
    C_hi, C_lo, fl = casc.casc_i8_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                              T(d["B_lo"]))
    torch.cuda.synchronize()
    C_hi, C_lo, fl = N(C_hi), N(C_lo), N(fl)
    rows = [0, m // 2, m - 1]
    c0, c1 = n - 96, n
    o_hi, o_lo, o_fl = orc.i8_casc_gemm(d["A_hi"][rows], d["A_lo"][rows],
                                        d["B_hi"][:, c0:c1].copy(), d["B_lo"][:, c0:c1].copy())
    assert bitwise(C_hi[rows, c0:c1], o_hi) and bitwise(C_lo[rows, c0:c1], o_lo)
    assert np.array_equal(fl[rows, c0:c1], o_fl)
    if variant == "b":
        assert fl.all()
        return
    rng = np.random.default_rng(cfg)
    ii = np.concatenate([rng.integers(0, m, 100), [0, m - 1]])
    jj = np.concatenate([rng.integers(0, n, 100), [n - 1, 0]])
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii, jj, C_hi, C_lo)
    assert np.max(np.abs(r["err"]) / orc.north_star_bound(k, r["absab"])) <= 1.0
    assert fl.sum() == 0


@pytest.mark.parametrize("world", [2, 3])
def test_i8_p_invariance_emulated_ranks(casc, world):
    """The INT8 multi-GPU data path rank by rank on one GPU: rank r packs its
    rows of A and its 256-column slab of B; the slabs concatenated in rank order
    are the all-gathered buffer; C is bitwise the single-call result."""
    import torch
    from paper_2303_04353_b200.multigpu import I8_BLOCK, col_slab, row_shard
    m, n, k = 300, 700, 530
    d = I.make_config(1, m=m, n=n, k=k, seed=13)
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    ref = [N(x) for x in casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)]
    blk = 2 * casc.casc_i8_packed_block_bytes(k)
    chunks = []
    for r in range(world):
        c0, c1, per = col_slab(n, world, r, I8_BLOCK)
        buf = torch.zeros(per * blk, dtype=torch.uint8, device="cuda")
        if c1 > c0:
            used = -(-(c1 - c0) // I8_BLOCK) * blk
            casc.casc_i8_pack(B_hi[:, c0:c1].contiguous(), B_lo[:, c0:c1].contiguous(), True,
                              packed=buf[:used])
        chunks.append(buf)
    pb = torch.cat(chunks)
    for r in range(world):
        r0, r1 = row_shard(m, world, r)
        pa = casc.casc_i8_pack(A_hi[r0:r1].contiguous(), A_lo[r0:r1].contiguous(), False)
        got = [N(x) for x in casc.casc_i8_gemm_packed(r1 - r0, n, k, pa, pb)]
        assert all(np.array_equal(g, x[r0:r1]) for g, x in zip(got, ref))


@pytest.mark.parametrize("m,n,k", [(600, 1, 300), (1, 700, 300), (257, 129, 8192),
                                   (70, 40, 16384 + 1)])
def test_i8_skinny_and_panel_edges(casc, orc, m, n, k):
    """One-column / one-row problems (raster with a single tile row or column),
    exactly one full 8192 panel, and two full panels plus one k."""
    d = I.make_config(1, m=m, n=n, k=k, seed=m + n)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo) and np.array_equal(fl, ofl)


@pytest.mark.parametrize("sa,sb,k", [(-700, -300, 500), (-760, -300, 500),
                                      (-775, -300, 8192 + 40), (-850, -300, 500)])
def test_i8_extreme_exponents(casc, orc, sa, sb, k):
    """Rows of A scaled by 2^sa and columns of B by 2^sb: products near 2^-1000
    (subnormal FP64x2 tails), near 2^-1060 (T.hi itself subnormal), around
    2^-1075 (partial underflow, two panels) and below 2^-1140 (everything rounds
    to signed zeros): bit-exact with the oracle (R25 rev. 2 rounding on the
    subnormal grid, signs of zero included)."""
    d = I.make_config(1, m=90, n=70, k=k, seed=31)
    for x in ("A_hi", "A_lo"):
        d[x] = np.ldexp(d[x], sa)
    for x in ("B_hi", "B_lo"):
        d[x] = np.ldexp(d[x], sb)
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    o_hi, o_lo, ofl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], 14)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo) and np.array_equal(fl, ofl)
    if sa + sb > -1100:
        assert np.all(np.abs(C_hi) < 2.0**(sa + sb + 20)) and np.any(C_hi != 0)


# ------------------------------------------------------------------ BLAS-style (NEXT-4)
@pytest.mark.parametrize("ta,tb,k", [("N", "N", 8192 + 300), ("T", "N", 8192 + 300),
                                     ("N", "T", 8192 + 300), ("T", "T", 8192 + 300),
                                     ("N", "N", 700), ("T", "T", 700)])
def test_i8_blas_ex_bit_exact(casc, orc, ta, tb, k):
    """casc_i8_gemm_fp64x2_ex: transposed operands, alpha / beta (reading R21)
    bit-exact with oracle.i8_casc_gemm_ex, with a two-panel k and ragged tiles
    and with a single panel (split mode: alpha / beta in the reduce kernel)."""
    import torch
    m, n = 130, 257
    d = I.make_config(1, m=m, n=n, k=k, seed=41)
    A = (d["A_hi"].T.copy(), d["A_lo"].T.copy()) if ta == "T" else (d["A_hi"], d["A_lo"])
    B = (d["B_hi"].T.copy(), d["B_lo"].T.copy()) if tb == "T" else (d["B_hi"], d["B_lo"])
    rng = np.random.default_rng(11)
    C0h = rng.uniform(-1, 1, (m, n))
    C0l = C0h * 2.0 ** -60 * rng.uniform(-1, 1, (m, n))
    for al, be in [((1.0, 0.0), (0.0, 0.0)), ((1.0 / 3.0, 2.0 ** -56), (0.0, 0.0)),
                   ((1.0, 0.0), (-0.7, 2.0 ** -60)), ((-4.0, 0.0), (1.5, 0.0))]:
        nan = be == (0.0, 0.0)  # beta = 0: C is not read (NaN in, finite out)
        C_hi = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda") if nan \
            else T(C0h)
        C_lo = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda") if nan \
            else T(C0l)
        fl = torch.empty((m, n), dtype=torch.uint8, device="cuda")
        casc.casc_i8_gemm_fp64x2_ex(ta, tb, al, T(A[0]), T(A[1]), T(B[0]), T(B[1]), be,
                                    C_hi, C_lo, flags=fl)
        o_hi, o_lo, o_fl = orc.i8_casc_gemm_ex(ta, tb, al, A[0], A[1], B[0], B[1], be,
                                               C0h.copy(), C0l.copy())
        assert bitwise(N(C_hi), o_hi) and bitwise(N(C_lo), o_lo), (ta, tb, al, be)
        assert np.array_equal(N(fl), o_fl)


def test_i8_blas_ex_degenerate(casc, orc):
    """k = 0 / alpha = 0: C := beta C and flags := 0 without reading A, B;
    strided C (ldc > n); workspace given explicitly; bad arguments rejected."""
    import torch
    m, n, k = 70, 90, 200
    rng = np.random.default_rng(5)
    C0 = rng.uniform(-1, 1, (m, n))
    be = (-0.7, 2.0 ** -60)
    C_hi, C_lo = T(C0), T(np.zeros((m, n)))
    fl = torch.full((m, n), 5, dtype=torch.uint8, device="cuda")
    casc.casc_i8_gemm_fp64x2_ex("N", "N", 0.0, None, None, None, None, be, C_hi, C_lo, flags=fl)
    o_hi, o_lo, _ = orc.i8_casc_gemm_ex("N", "N", (0.0, 0.0), np.zeros((m, 0)), np.zeros((m, 0)),
                                        np.zeros((0, n)), np.zeros((0, n)), be, C0.copy(),
                                        np.zeros((m, n)))
    assert bitwise(N(C_hi), o_hi) and bitwise(N(C_lo), o_lo) and N(fl).sum() == 0
    # strided C inside a wider buffer, explicit workspace, y = 8
    d = I.make_config(2, m=m, n=n, k=k, seed=43)
    big_h = T(np.tile(C0, (1, 2)))
    big_l = T(np.zeros((m, 2 * n)))
    ws = torch.empty(casc.casc_i8_workspace_bytes(m, n, k, 8), dtype=torch.uint8, device="cuda")
    casc.casc_i8_gemm_fp64x2_ex("N", "N", 2.0, T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                T(d["B_lo"]), 1.0, big_h[:, :n], big_l[:, :n], y=8,
                                workspace=ws)
    o_hi, o_lo, _ = orc.i8_casc_gemm_ex("N", "N", (2.0, 0.0), d["A_hi"], d["A_lo"], d["B_hi"],
                                        d["B_lo"], (1.0, 0.0), C0.copy(), np.zeros((m, n)), y=8)
    assert bitwise(N(big_h[:, :n]).copy(), o_hi) and bitwise(N(big_l[:, :n]).copy(), o_lo)
    assert np.array_equal(N(big_h[:, n:]), C0)  # untouched
    with pytest.raises(casc.CascError):
        casc.casc_i8_gemm_fp64x2_ex("N", "N", 1.0, T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                    T(d["B_lo"]), 0.0, T(C0), T(C0), y=2)


# ------------------------------------------------------------------ host operands
@pytest.mark.parametrize("m,n,k,slab,scol,y", [(700, 300, 900, 256, 256, 14),
                                               (300, 257, 8192 + 100, 0, 0, 14),
                                               (513, 700, 640, 256, 256, 9)])
def test_i8_host_operands_bitwise(casc, m, n, k, slab, scol, y):
    """casc_i8_gemm_fp64x2_host (blocks of 256-multiple row and column slabs
    streamed from pinned host memory): bitwise the device-resident
    casc_i8_gemm_fp64x2 result."""
    import torch
    d = I.make_config(2, m=m, n=n, k=k, seed=61)
    ref = gpu_gemm(casc, d, y=y)
    P = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    C_hi, C_lo, fl = casc.casc_i8_gemm_fp64x2_host(P(d["A_hi"]), P(d["A_lo"]), P(d["B_hi"]),
                                                   P(d["B_lo"]), y=y, slab_rows=slab,
                                                   slab_cols=scol)
    assert bitwise(C_hi.numpy(), ref[0]) and bitwise(C_lo.numpy(), ref[1])
    assert np.array_equal(fl.numpy(), ref[2])


# ------------------------------------------------------------------ split mode
@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (512, 300, 700), (256, 128, 8192),
                                   (700, 520, 1000), (130, 257, 300)])
def test_i8_split_mode_bitwise(casc, orc, m, n, k):
    """Small single-panel problems run one work item per (tile, k-block part)
    and sum the parts' exact partial products in a reduce kernel (R25 rev. 2
    rounds the exact sum, so any partition is bitwise the same): split and
    unsplit runs agree bitwise, and both match the oracle on sampled rows."""
    import os
    d = I.make_config(1, m=m, n=n, k=k, seed=81)
    split = gpu_gemm(casc, d)
    os.environ["CASC_I8_SPLIT"] = "0"
    try:
        whole = gpu_gemm(casc, d)
    finally:
        del os.environ["CASC_I8_SPLIT"]
    for a, b in zip(split, whole):
        assert np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                              np.ascontiguousarray(b).view(np.uint8))
    rows = np.unique(np.linspace(0, m - 1, 6).astype(int))
    o_hi, o_lo, o_fl = orc.i8_casc_gemm(d["A_hi"][rows], d["A_lo"][rows], d["B_hi"], d["B_lo"])
    assert bitwise(split[0][rows], o_hi) and bitwise(split[1][rows], o_lo)
    assert np.array_equal(split[2][rows], o_fl)


def test_i8_rounding_ties_and_near_ties(casc, orc):
    """Panel values whose exact product sits exactly halfway between two
    doubles (at T.hi's and at T.lo's rounding position) or one unit of the
    fixed-point grid away from it: the kernel's integer rounding (R25 rev. 2,
    the 128-bit fast path) must pick the same neighbour as the oracle's big
    integer rounding, bit for bit."""
    rng = np.random.default_rng(17)
    m, n = 40, 36
    A_hi = np.zeros((m, 1))
    B_hi = np.zeros((1, n))
    # (1 + a 2^-26)(1 + b 2^-27) = 1 + a 2^-26 + b 2^-27 + ab 2^-53: ties at the
    # 2^-53 position for odd ab, different parities of the kept part
    for i in range(m):
        A_hi[i, 0] = (1.0 + float(rng.integers(1, 2**20)) * 2.0**-46) * (-1.0) ** i
    for j in range(n):
        B_hi[0, j] = 1.0 + float(rng.integers(1, 2**20)) * 2.0**-47
    A_hi[::3, 0] = 1.0 + 2.0**-26
    B_hi[0, ::4] = 1.0 + 2.0**-27
    A_lo = np.zeros_like(A_hi)
    B_lo = np.zeros_like(B_hi)
    A_lo[1::5, 0] = 2.0**-60  # ties at the lo position too
    B_lo[0, 2::5] = -(2.0**-61)
    d = {"A_hi": A_hi, "A_lo": A_lo, "B_hi": B_hi, "B_lo": B_lo}
    C_hi, C_lo, fl = gpu_gemm(casc, d)
    o_hi, o_lo, o_fl = orc.i8_casc_gemm(A_hi, A_lo, B_hi, B_lo)
    assert bitwise(C_hi, o_hi) and bitwise(C_lo, o_lo) and np.array_equal(fl, o_fl)
    # the products really are DD-exact here: C_hi + C_lo == the exact product
    from fractions import Fraction as F
    for i in range(0, m, 7):
        for j in range(0, n, 5):
            ex = (F(A_hi[i, 0]) + F(A_lo[i, 0])) * (F(B_hi[0, j]) + F(B_lo[0, j]))
            err = abs(F(C_hi[i, j]) + F(C_lo[i, j]) - ex)
            assert err <= abs(ex) * F(2) ** -104


# ------------------------------------------------------------------ SYRK (NEXT-4)
@pytest.mark.parametrize("uplo,trans,n,k,al,be", [
    ("L", "N", 300, 700, (1.0, 0.0), (0.0, 0.0)), ("U", "N", 520, 8192 + 100, (1.0, 0.0), (0.0, 0.0)),
    ("L", "T", 257, 300, (1.0 / 3.0, 2.0 ** -56), (-0.7, 2.0 ** -60)),
    ("U", "T", 64, 64, (2.0, 0.0), (1.0, 0.0))])
def test_i8_syrk_bit_exact(casc, orc, uplo, trans, n, k, al, be):
    """casc_i8_syrk_fp64x2 (triangular pair-tile list): bit-exact with the
    oracle's triangle, the other triangle and its flags untouched."""
    import torch
    d = I.make_config(2, m=n, n=k, k=k, seed=97)
    A_hi, A_lo = d["A_hi"][:n, :k], d["A_lo"][:n, :k]
    Ast = (A_hi.T.copy(), A_lo.T.copy()) if trans == "T" else (A_hi.copy(), A_lo.copy())
    rng = np.random.default_rng(3)
    C0 = rng.uniform(-1, 1, (n, n))
    C_hi, C_lo = T(C0), T(np.zeros((n, n)))
    fl = torch.full((n, n), 9, dtype=torch.uint8, device="cuda")
    casc.casc_i8_syrk_fp64x2(uplo, trans, al, T(Ast[0]), T(Ast[1]), be, C_hi, C_lo, flags=fl)
    o_hi, o_lo, o_fl = orc.i8_casc_syrk(uplo, trans, al, *Ast, be, C0, np.zeros((n, n)),
                                        np.full((n, n), 9, np.uint8))
    assert bitwise(N(C_hi), o_hi) and bitwise(N(C_lo), o_lo) and np.array_equal(N(fl), o_fl)


# ------------------------------------------------------------------ TRSM (NEXT-4)
@pytest.mark.parametrize("uplo,trans,diag,m,n", [("L", "N", "N", 300, 40), ("U", "N", "U", 520, 9),
                                                 ("L", "T", "N", 600, 17), ("U", "T", "N", 256, 5),
                                                 ("L", "N", "N", 1100, 6), ("U", "T", "N", 1300, 3)])
def test_i8_trsm_bit_exact(casc, orc, uplo, trans, diag, m, n):
    """casc_i8_trsm_fp64x2 (reading R27 with the INT8 cascade as the GEMM):
    bit-exact with orc_i8_casc_trsm (diagonal inverses bitwise, INT8 GEMMs
    bit-exact), alpha = 2^p included."""
    rng = np.random.default_rng(29)
    A_hi = rng.uniform(-1, 1, (m, m)) / m
    A_hi = np.tril(A_hi) if uplo == "L" else np.triu(A_hi)
    A_lo = A_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, m))
    dgl = 1.0 + rng.uniform(0, 1, m)
    A_hi[np.arange(m), np.arange(m)] = dgl
    A_lo[np.arange(m), np.arange(m)] = dgl * 2.0 ** -55
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    for al in ((1.0, 0.0), (4.0, 0.0)):
        Xh, Xl = T(B_hi), T(B_lo)
        casc.casc_i8_trsm_fp64x2(uplo, diag, al, T(A_hi), T(A_lo), Xh, Xl, trans=trans)
        o_hi, o_lo = orc.i8_casc_trsm(uplo, diag, al, A_hi, A_lo, B_hi, B_lo, trans=trans)
        assert bitwise(N(Xh), o_hi) and bitwise(N(Xl), o_lo), al
