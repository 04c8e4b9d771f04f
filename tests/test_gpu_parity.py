"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE north star):
  * split slices and scale exponents: bit-exact (values, +-0 equal);
  * bins 0-2 of every panel: bit-exact (they are exact);
  * bin 3-6: within gamma_{4k+1} sum|terms| of its exact value (order differs,
    DESIGN.md reading R17);
  * epilogue: C equals the oracle's combine applied to the GPU's own bins,
    bit for bit (same DD algorithm, reading R9);
  * final C: |C_gpu - C*| <= 4 k 2^-104 (|A||B|)_ij for every checked entry;
  * flags identical to the oracle's.
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


def run(casc, d, **kw):
    return [N(x) if x is not None else None
            for x in casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                           T(d["B_lo"]), **kw)]


def same_values(x, y):
    return bool(np.all((x == y) | (np.isnan(x) & np.isnan(y))))


SHAPES = [(0, 64, 64, 64), (1, 77, 70, 600), (2, 96, 130, 513), (1, 1, 1, 1), (1, 3, 5, 9),
          (1, 65, 129, 257), (1, 128, 64, 256)]


# ------------------------------------------------------------------ split a2-a4
@pytest.mark.parametrize("cfg,m,n,k", SHAPES)
def test_split_bit_exact(casc, orc, cfg, m, n, k):
    d = I.make_config(cfg, m=m, n=n, k=k)
    SA, e = casc.casc_split_a(T(d["A_hi"]), T(d["A_lo"]))
    SB, f = casc.casc_split_b(T(d["B_hi"]), T(d["B_lo"]))
    SA, e, SB, f = N(SA), N(e), N(SB), N(f)
    c = orc.select_widths(k)
    assert casc.casc_select_widths(k) == c
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        oa, oe = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        ob, of = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        assert np.array_equal(e[q], oe) and np.array_equal(f[q], of)
        assert same_values(SA[:, :, p0:p1], oa)
        assert same_values(SB[:, p0:p1, :], ob)


def test_split_full_mantissa(casc, orc):
    """Leading zeros / slice-3 rounding (full-mantissa set)."""
    hi, lo = I.full_mantissa(3, 40, 520)
    SA, e = casc.casc_split_a(T(hi), T(lo))
    SB, f = casc.casc_split_b(T(hi.T.copy()), T(lo.T.copy()))
    SA, e, SB, f = N(SA), N(e), N(SB), N(f)
    c = orc.select_widths(520)
    for q, p0 in enumerate(range(0, 520, 256)):
        p1 = min(520, p0 + 256)
        oa, oe = orc.split_a_panel(hi[:, p0:p1], lo[:, p0:p1], c)
        assert np.array_equal(e[q], oe) and same_values(SA[:, :, p0:p1], oa)
        ob, of = orc.split_b_panel(hi.T[p0:p1].copy(), lo.T[p0:p1].copy(), c)
        assert np.array_equal(f[q], of) and same_values(SB[:, p0:p1, :], ob)


# ------------------------------------------------------------------ bins a5
@pytest.mark.parametrize("cfg,m,n,k", SHAPES[:6])
def test_bins_bit_exact_and_bin36_bound(casc, orc, cfg, m, n, k):
    d = I.make_config(cfg, m=m, n=n, k=k)
    c = orc.select_widths(k)
    f36 = 2.0 ** (c[2] - c[0])
    u = 2.0**-53
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        kp = p1 - p0
        gb = N(casc.casc_debug_bins(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]), q))
        oa, _ = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        ob, _ = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        obins = orc.panel_bins(oa, ob, c)
        for b in range(3):
            assert same_values(gb[b], obins[b]), f"bin {b} panel {q}"
        # bin 3-6: gamma bound around the exact value of the same terms
        x = np.concatenate([oa[0], f36 * oa[1], f36 * oa[2], oa[3]], axis=1)  # m x 4kp
        y = np.concatenate([ob[3], ob[4], ob[5], ob[6]], axis=0)              # 4kp x n
        absterms = np.abs(x) @ np.abs(y)
        gamma = (4 * kp + 1) * u / (1 - (4 * kp + 1) * u)
        for i in range(0, m, max(1, m // 9)):
            for j in range(0, n, max(1, n // 7)):
                eh, el = orc.exact_dot(x[i], y[:, j])
                err = abs((gb[3, i, j] - eh) - el)
                assert err <= gamma * absterms[i, j] * (1 + 1e-12) + 1e-300
                assert abs(gb[3, i, j] - obins[3, i, j]) <= 2 * gamma * absterms[i, j] * (1 + 1e-12)


# ------------------------------------------------------------------ combine a6
@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 33, 40, 700), (2, 70, 66, 300)])
def test_epilogue_bitwise_on_gpu_bins(casc, orc, cfg, m, n, k):
    """C_gpu == oracle combine + FP64x2 panel accumulation of the GPU's own bins."""
    d = I.make_config(cfg, m=m, n=n, k=k)
    c = orc.select_widths(k)
    C_hi, C_lo, flags = run(casc, d)
    ref_hi = np.zeros((m, n))
    ref_lo = np.zeros((m, n))
    ref_fl = np.zeros((m, n), dtype=np.uint8)
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        gb = N(casc.casc_debug_bins(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]), q))
        _, e = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        _, f = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        for i in range(m):
            for j in range(n):
                th, tl = orc.combine(gb[0, i, j], gb[1, i, j], gb[2, i, j], gb[3, i, j],
                                     int(e[i]) + int(f[j]), c)
                ref_hi[i, j], ref_lo[i, j] = orc.dd_add(ref_hi[i, j], ref_lo[i, j], th, tl)
                ref_fl[i, j] |= gb[0, i, j] == 0.0
    assert same_values(C_hi, ref_hi) and same_values(C_lo, ref_lo)
    assert np.array_equal(flags, ref_fl)


# ------------------------------------------------------------------ final C
def _exact_check(orc, d, C_hi, C_lo, ii, jj):
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii, jj, C_hi, C_lo)
    bound = orc.north_star_bound(d["k"], r["absab"])
    return np.max(np.abs(r["err"]) / np.maximum(bound, 1e-300))


@pytest.mark.parametrize("cfg,m,n,k", SHAPES)
def test_final_c_within_bound_and_flags(casc, orc, cfg, m, n, k):
    d = I.make_config(cfg, m=m, n=n, k=k)
    C_hi, C_lo, flags = run(casc, d)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    assert _exact_check(orc, d, C_hi, C_lo, ii.ravel(), jj.ravel()) <= 1.0
    o_hi, o_lo, o_fl = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    assert np.array_equal(flags, o_fl)
    # both within the bound of C*, hence within twice the bound of each other
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel())
    diff = np.abs((C_hi - o_hi) + (C_lo - o_lo)).ravel()
    assert np.all(diff <= 2 * orc.north_star_bound(k, r["absab"]))


def test_cfg1_full_size_sampled(casc, orc):
    """cfg1 (1024^3) at full size: sampled exact entries, plus whole-row oracle
    parity of flags and C for a few rows."""
    d = I.make_config(1)
    C_hi, C_lo, flags = run(casc, d)
    rng = np.random.default_rng(0)
    ii = rng.integers(0, 1024, 3000)
    jj = rng.integers(0, 1024, 3000)
    assert _exact_check(orc, d, C_hi, C_lo, ii, jj) <= 1.0
    rows = [0, 511, 1023]
    sub = dict(d, A_hi=d["A_hi"][rows], A_lo=d["A_lo"][rows], m=3)
    o_hi, o_lo, o_fl = orc.casc_gemm(sub["A_hi"], sub["A_lo"], d["B_hi"], d["B_lo"])
    assert np.array_equal(flags[rows], o_fl) and flags.sum() == 0


def test_cancellation_configs(casc, orc):
    """cfg3 structure (reading R13) at 256 x 256 x 4096: 3a and 3c raise no flags
    and stay within the bound; 3b flags every entry; flags == oracle's."""
    for variant in ("a", "b", "c"):
        d = I.make_config(3, m=256, n=256, k=4096, variant=variant)
        C_hi, C_lo, flags = run(casc, d)
        rows = [0, 100, 255]
        o_hi, o_lo, o_fl = orc.casc_gemm(d["A_hi"][rows], d["A_lo"][rows], d["B_hi"], d["B_lo"])
        assert np.array_equal(flags[rows], o_fl)
        if variant == "b":
            assert flags.all()
        else:
            assert flags.sum() == 0
            rng = np.random.default_rng(1)
            ii, jj = rng.integers(0, 256, 400), rng.integers(0, 256, 400)
            assert _exact_check(orc, d, C_hi, C_lo, ii, jj) <= 1.0


def test_worst_case_flagged(casc):
    """§3.6 worst case through the GPU: bin 0 == 0 -> flagged."""
    import torch
    A_hi = torch.tensor([[1.0, 2.0**-100]], dtype=torch.float64).cuda()
    A_lo = torch.zeros_like(A_hi)
    B_hi = torch.tensor([[0.0], [1.0]], dtype=torch.float64).cuda()
    B_lo = torch.zeros_like(B_hi)
    C_hi, C_lo, fl = casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)
    assert fl.item() == 1 and C_hi.item() == 2.0**-100 and C_lo.item() == 0.0


def test_edge_cases(casc):
    import torch
    z = lambda *s: torch.zeros(s, dtype=torch.float64, device="cuda")
    # m == 0 / n == 0: no-op
    C = casc.casc_gemm_fp64x2(z(0, 5), z(0, 5), z(5, 3), z(5, 3))
    assert C[0].shape == (0, 3)
    # k == 0: C := 0, flags := 0 (reading R18)
    C_hi = torch.full((4, 3), 7.0, dtype=torch.float64, device="cuda")
    C_lo = torch.full((4, 3), 7.0, dtype=torch.float64, device="cuda")
    fl = torch.full((4, 3), 9, dtype=torch.uint8, device="cuda")
    casc.casc_gemm_fp64x2(z(4, 0), z(4, 0), z(0, 3), z(0, 3), C_hi=C_hi, C_lo=C_lo, flags=fl)
    assert C_hi.abs().sum().item() == 0 and C_lo.abs().sum().item() == 0 and fl.sum().item() == 0
    # zero rows of A -> zero C rows, flagged
    d = I.make_config(1, m=20, n=20, k=300, seed=4)
    d["A_hi"][5] = 0.0
    d["A_lo"][5] = 0.0
    C_hi, C_lo, flags = run(casc, d)
    assert np.all(C_hi[5] == 0) and np.all(C_lo[5] == 0) and np.all(flags[5] == 1)
    assert flags.sum() == 20
    # aliasing C with A is rejected
    A = torch.rand(8, 8, dtype=torch.float64, device="cuda")
    with pytest.raises(casc.CascError):
        casc.casc_gemm_fp64x2(A, A, A, A, C_hi=A, C_lo=z(8, 8))


def test_strided_inputs_and_outputs(casc, orc):
    """Leading dimensions > width on A, B and C."""
    import torch
    d = I.make_config(1, m=40, n=36, k=300, seed=6)
    big = lambda a, extra: torch.from_numpy(np.pad(a, ((0, 0), (0, extra)))).cuda()
    A_hi, A_lo = big(d["A_hi"], 5)[:, :300], big(d["A_lo"], 5)[:, :300]
    B_hi, B_lo = big(d["B_hi"], 3)[:, :36], big(d["B_lo"], 3)[:, :36]
    Cb_hi = torch.zeros((40, 41), dtype=torch.float64, device="cuda")
    Cb_lo = torch.zeros((40, 41), dtype=torch.float64, device="cuda")
    casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=Cb_hi[:, :36], C_lo=Cb_lo[:, :36])
    ref = run(casc, d)
    assert same_values(N(Cb_hi)[:, :36], ref[0]) and same_values(N(Cb_lo)[:, :36], ref[1])
    assert np.all(N(Cb_hi)[:, 36:] == 0)


def test_determinism_and_scaling_neutrality(casc):
    d = I.make_config(1, m=200, n=190, k=777, seed=3)
    s = I.make_config(2, m=200, n=190, k=777, seed=3)
    r1 = run(casc, d)
    r2 = run(casc, d)
    assert all(np.array_equal(a, b) for a, b in zip(r1, r2))
    rs = run(casc, s)
    u = I.int_uniform(3, I.STREAM_ROW_EXP, 200, -30, 30)
    v = I.int_uniform(3, I.STREAM_COL_EXP, 190, -30, 30)
    sc = np.ldexp(1.0, u[:, None] + v[None, :])
    assert np.array_equal(r1[0] * sc, rs[0]) and np.array_equal(r1[1] * sc, rs[1])
    assert np.array_equal(r1[2], rs[2])


def test_workspace_and_packed_paths_agree(casc):
    import torch
    d = I.make_config(1, m=130, n=200, k=515, seed=8)
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    r0 = casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)
    ws = torch.empty(casc.casc_workspace_bytes(130, 200, 515), dtype=torch.uint8, device="cuda")
    r1 = casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, workspace=ws)
    pa = casc.casc_pack_a(A_hi, A_lo)
    pb = casc.casc_pack_b(B_hi, B_lo)
    r2 = casc.casc_gemm_packed(130, 200, 515, pa, pb)
    for x, y in ((r0, r1), (r0, r2)):
        assert all(torch.equal(a, b) for a, b in zip(x, y))


def test_column_slab_packing_is_blockwise(casc):
    """Packing a 64-multiple column slab of B gives exactly the corresponding
    byte range of the full packed B (the multi-GPU all-gather premise)."""
    import torch
    d = I.make_config(4, m=64, n=256, k=300)
    B_hi, B_lo = T(d["B_hi"]), T(d["B_lo"])
    full = casc.casc_pack_b(B_hi, B_lo)
    blk = casc.casc_packed_b_block_bytes(300)
    for r in range(4):
        part = casc.casc_pack_b(B_hi[:, 64 * r:64 * (r + 1)], B_lo[:, 64 * r:64 * (r + 1)])
        assert torch.equal(part, full[r * blk:(r + 1) * blk])


# ------------------------------------------------------------------ full sizes
def _sub_oracle(orc, d, rows, c0, c1):
    """ORACLE-CASCADE on rows x [c0, c1): columns are independent (per-column
    scales), so this equals the same block of the full oracle result."""
    return orc.casc_gemm(d["A_hi"][rows], d["A_lo"][rows], d["B_hi"][:, c0:c1].copy(),
                         d["B_lo"][:, c0:c1].copy())


@pytest.mark.parametrize("cfg,variant", [(2, "a"), (3, "a"), (4, "a")])
def test_full_size_configs_sampled(casc, orc, cfg, variant):
    """BASELINE configs 2, 3 and 4 at FULL size through casc_gemm_fp64x2 (the
    kernels and launch configuration bench.py times): sampled entries vs the
    exact product (north-star bound), and a row x column block vs ORACLE-CASCADE
    (flags identical, C within twice the bound)."""
    import torch
    d = I.make_config(cfg, variant=variant)
    m, n, k = d["m"], d["n"], d["k"]
    C_hi, C_lo, flags = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                              T(d["B_lo"]))
    torch.cuda.synchronize()
    rng = np.random.default_rng(cfg)
    ii = np.concatenate([rng.integers(0, m, 120), [0, m - 1]])
    jj = np.concatenate([rng.integers(0, n, 120), [n - 1, 0]])
    C_hi, C_lo, flags = N(C_hi), N(C_lo), N(flags)
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii, jj, C_hi, C_lo)
    assert np.max(np.abs(r["err"]) / orc.north_star_bound(k, r["absab"])) <= 1.0
    rows = [0, m // 2, m - 1]
    c0, c1 = n - 96, n
    o_hi, o_lo, o_fl = _sub_oracle(orc, d, rows, c0, c1)
    assert np.array_equal(flags[rows, c0:c1], o_fl)
    rr = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"],
                           np.repeat(rows, c1 - c0), np.tile(np.arange(c0, c1), len(rows)))
    diff = np.abs((C_hi[rows, c0:c1] - o_hi) + (C_lo[rows, c0:c1] - o_lo)).ravel()
    assert np.all(diff <= 2 * orc.north_star_bound(k, rr["absab"]))
    assert flags.sum() == 0


@pytest.mark.parametrize("cfg,variant", [(2, "a"), (3, "a"), (4, "a")])
def test_full_size_exact_lines(casc, orc, cfg, variant):
    """BASELINE configs 2, 3 and 4 at FULL size, as bench.py launches them:
    EVERY entry of one row (full for cfg2 / cfg3; its first 2048 columns for
    cfg4), one full column (cfg2) and a 64 x 128 block of C against the exact
    product (oracle/exact_fixed.py, k in exact chunks) within the north-star
    bound, and the row against ORACLE-CASCADE (flags identical, C within twice
    the bound).  (A full cfg4 row or column costs the exact evaluator ~1.5 min
    of host time: the digits of all of B or A.)"""
    import torch
    from oracle import exact_fixed as EF
    d = I.make_config(cfg, variant=variant)
    m, n, k = d["m"], d["n"], d["k"]
    C_hi, C_lo, flags = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                              T(d["B_lo"]))
    torch.cuda.synchronize()
    C_hi, C_lo, flags = N(C_hi), N(C_lo), N(flags)
    rng = np.random.default_rng(100 + cfg)
    i, j = int(rng.integers(0, m)), int(rng.integers(0, n))
    b0, b1 = int(rng.integers(0, m - 64)), int(rng.integers(0, n - 128))
    absA = np.abs(d["A_hi"]) + np.abs(d["A_lo"])
    absB = np.abs(d["B_hi"]) + np.abs(d["B_lo"])
    rn = 2048 if cfg == 4 else n
    lines = [(slice(i, i + 1), slice(0, rn)), (slice(b0, b0 + 64), slice(b1, b1 + 128))]
    if cfg == 2:
        lines.append((slice(0, m), slice(j, j + 1)))
    for rows, cols in lines:
        Bh = np.ascontiguousarray(d["B_hi"][:, cols])
        Bl = np.ascontiguousarray(d["B_lo"][:, cols])
        err, _ = EF.errors(d["A_hi"][rows], d["A_lo"][rows], Bh, Bl, C_hi[rows, cols],
                           C_lo[rows, cols])
        bound = orc.north_star_bound(k, (absA[rows] @ absB[:, cols]) * (1 - 2.0 ** -40))
        assert np.all(np.abs(err) <= bound), (rows, cols)
    o_hi, o_lo, o_fl = _sub_oracle(orc, d, [i], 0, rn)
    assert np.array_equal(flags[[i], :rn], o_fl)
    diff = np.abs((C_hi[[i], :rn] - o_hi) + (C_lo[[i], :rn] - o_lo))
    assert np.all(diff <= 2 * orc.north_star_bound(k, absA[[i]] @ absB[:, :rn]))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_p_invariance_emulated_ranks(casc, world):
    """The multi-GPU data path run rank by rank on one GPU (no collective is
    needed to emulate it: rank r packs its rows of A and its column slab of B;
    the packed slabs concatenated in rank order are the all-gathered buffer):
    C is bitwise identical to the single-call result for any world size."""
    import torch
    from paper_2303_04353_b200.multigpu import col_slab, row_shard
    m, n, k = 300, 700, 530
    d = I.make_config(1, m=m, n=n, k=k, seed=13)
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    ref = casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo)
    blk = casc.casc_packed_b_block_bytes(k)
    chunks = []
    for r in range(world):
        c0, c1, per = col_slab(n, world, r)
        buf = torch.zeros(per * blk, dtype=torch.uint8, device="cuda")
        if c1 > c0:
            used = -(-(c1 - c0) // 64) * blk
            casc.casc_pack_b(B_hi[:, c0:c1], B_lo[:, c0:c1], packed=buf[:used])
        chunks.append(buf)
    pb = torch.cat(chunks)
    for r in range(world):
        r0, r1 = row_shard(m, world, r)
        pa = casc.casc_pack_a(A_hi[r0:r1], A_lo[r0:r1])
        out = casc.casc_gemm_packed(r1 - r0, n, k, pa, pb)
        for x, y in zip(out, ref):
            assert torch.equal(x, y[r0:r1])


# ------------------------------------------------------------------ simple path (NEXT-2)
EXACT_PRODUCTS = [(0, 0), (0, 1), (1, 0), (0, 2), (1, 1), (2, 0)]
ROUNDED_PRODUCTS = [(0, 3), (1, 4), (2, 5), (3, 6)]


@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 70, 90, 600), (2, 65, 33, 300)])
def test_slice_products(casc, orc, cfg, m, n, k):
    """Every slice GEMM of the simple path: the six exact products of
    eqn:Gemm10 equal the exact sums bit for bit (BASELINE north star "match
    bit-exactly on each slice-GEMM wherever the digit budgets make FP64
    accumulation exact"); the four others are within gamma_{k+1} sum|terms|."""
    d = I.make_config(cfg, m=m, n=n, k=k)
    c = orc.select_widths(k)
    A = [T(d[x]) for x in ("A_hi", "A_lo")]
    B = [T(d[x]) for x in ("B_hi", "B_lo")]
    u = 2.0**-53
    for q, p0 in enumerate(range(0, k, 256)):
        p1 = min(k, p0 + 256)
        oa, _ = orc.split_a_panel(d["A_hi"][:, p0:p1], d["A_lo"][:, p0:p1], c)
        ob, _ = orc.split_b_panel(d["B_hi"][p0:p1], d["B_lo"][p0:p1], c)
        for sa, sb in EXACT_PRODUCTS + ROUNDED_PRODUCTS:
            P = N(casc.casc_slice_product(*A, *B, sa, sb, q))
            rows = range(0, m, max(1, m // 6))
            cols = range(0, n, max(1, n // 5))
            for i in rows:
                for j in cols:
                    eh, el = orc.exact_dot(oa[sa][i], ob[sb][:, j])
                    if (sa, sb) in EXACT_PRODUCTS:
                        assert el == 0.0 and P[i, j] == eh, (sa, sb, i, j)
                    else:
                        bound = (p1 - p0 + 1) * u * float(np.abs(oa[sa][i]) @ np.abs(ob[sb][:, j]))
                        assert abs((P[i, j] - eh) - el) <= bound * (1 + 1e-12)
            if (sa, sb) in EXACT_PRODUCTS:  # all entries: any exact evaluation agrees
                assert np.array_equal(P, oa[sa] @ ob[sb])


@pytest.mark.parametrize("cfg,m,n,k", [(0, 64, 64, 64), (1, 77, 70, 600), (2, 96, 130, 513),
                                       (3, 64, 64, 1024)])
def test_simple_path_agrees_with_fused(casc, orc, cfg, m, n, k):
    """§4.2 simple path vs the fused kernel: identical flags, C within twice the
    north-star bound of each other (both within it of C*)."""
    d = I.make_config(cfg, m=m, n=n, k=k, variant="b") if cfg == 3 else \
        I.make_config(cfg, m=m, n=n, k=k)
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    s_hi, s_lo, s_fl = (N(x) for x in casc.casc_gemm_fp64x2_simple(*args))
    f_hi, f_lo, f_fl = (N(x) for x in casc.casc_gemm_fp64x2(*args))
    assert np.array_equal(s_fl, f_fl)
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel(),
                          s_hi, s_lo)
    bound = orc.north_star_bound(k, r["absab"])
    if cfg != 3:
        assert np.all(np.abs(r["err"]) <= bound)
        diff = np.abs((s_hi - f_hi) + (s_lo - f_lo)).ravel()
        assert np.all(diff <= 2 * bound)
    else:
        assert s_fl.all()


# ------------------------------------------------------------------ BLAS-style (NEXT-4)
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_blas_ex_transposes_bitwise(casc, ta, tb):
    """op(X) = X^T changes only how the split kernels read: the result is bitwise
    the non-transposed product (alpha = 1, beta = 0)."""
    import torch
    m, n, k = 70, 90, 300
    d = I.make_config(1, m=m, n=n, k=k, seed=23)
    ref = run(casc, d)
    A = (d["A_hi"].T.copy(), d["A_lo"].T.copy()) if ta == "T" else (d["A_hi"], d["A_lo"])
    B = (d["B_hi"].T.copy(), d["B_lo"].T.copy()) if tb == "T" else (d["B_hi"], d["B_lo"])
    C_hi = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")  # beta=0: unread
    C_lo = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    fl = torch.empty((m, n), dtype=torch.uint8, device="cuda")
    casc.casc_gemm_fp64x2_ex(ta, tb, 1.0, T(A[0]), T(A[1]), T(B[0]), T(B[1]), 0.0, C_hi, C_lo,
                             flags=fl)
    assert same_values(N(C_hi), ref[0]) and same_values(N(C_lo), ref[1])
    assert np.array_equal(N(fl), ref[2])


def test_blas_ex_alpha_beta(casc, orc):
    """C := alpha P + beta C: bitwise equal to the oracle's FP64x2 update applied
    to the GPU's own product P (reading R21), and within the bound of the exact
    alpha A B + beta C; alpha = 0 / k = 0 give beta C without touching A, B."""
    import torch
    m, n, k = 65, 129, 513
    d = I.make_config(2, m=m, n=n, k=k, seed=29)
    P_hi, P_lo, P_fl = run(casc, d)
    rng = np.random.default_rng(7)
    C0 = rng.uniform(-1, 1, (m, n))
    al, be = (1.0 / 3.0, 2.0 ** -56), (-0.7, 2.0 ** -60)
    C_hi, C_lo = T(C0), T(np.zeros((m, n)))
    casc.casc_gemm_fp64x2_ex("N", "N", al, T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                             T(d["B_lo"]), be, C_hi, C_lo)
    g_hi, g_lo = N(C_hi), N(C_lo)
    for i in range(0, m, 7):
        for j in range(0, n, 11):
            th, tl = orc.dd_mul(al[0], al[1], P_hi[i, j], P_lo[i, j])
            uh, ul = orc.dd_mul(be[0], be[1], C0[i, j], 0.0)
            th, tl = orc.dd_add(th, tl, uh, ul)
            assert (g_hi[i, j], g_lo[i, j]) == (th, tl)
    # vs the oracle's full BLAS update (bin 3-6 order differs: bound, not bits)
    o_hi, o_lo, o_fl = orc.casc_gemm_ex("N", "N", al, d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"],
                                        be, C0, np.zeros((m, n)))
    ii, jj = np.meshgrid(np.arange(m), np.arange(n), indexing="ij")
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii.ravel(), jj.ravel())
    bound = (abs(al[0]) * 2 * orc.north_star_bound(k, r["absab"])).reshape(m, n) \
        + 2.0 ** -100 * (np.abs(g_hi))
    assert np.all(np.abs((g_hi - o_hi) + (g_lo - o_lo)) <= bound)
    # alpha == 0 and k == 0: C := beta C, flags := 0
    C_hi, C_lo = T(C0), T(np.zeros((m, n)))
    fl = torch.full((m, n), 5, dtype=torch.uint8, device="cuda")
    casc.casc_gemm_fp64x2_ex("N", "N", 0.0, None, None, None, None, be, C_hi, C_lo, flags=fl)
    for i in range(0, m, 9):
        for j in range(0, n, 13):
            assert (N(C_hi)[i, j], N(C_lo)[i, j]) == orc.dd_mul(be[0], be[1], C0[i, j], 0.0)
    assert N(fl).sum() == 0


@pytest.mark.parametrize("m,n,k", [(1024, 1024, 1024), (200, 300, 700), (64, 64, 600)])
def test_split_mode_bitwise(casc, m, n, k):
    """Small problems run one work item per (tile, panel) plus an ordered FP64x2
    reduction (casc_api.cu split_plan); the result must be bitwise the
    one-item-per-tile result (same additions in the same order)."""
    import os
    d = I.make_config(1, m=m, n=n, k=k, seed=31)
    args = [T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    split = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    os.environ["CASC_SPLIT_MODE"] = "0"
    try:
        whole = [N(x) for x in casc.casc_gemm_fp64x2(*args)]
    finally:
        del os.environ["CASC_SPLIT_MODE"]
    for a, b in zip(split, whole):
        assert np.array_equal(a, b)
    # with alpha / beta through the reduction kernel as well
    al, be = (0.75, 2.0**-60), (1.5, 0.0)
    C0 = np.random.default_rng(3).uniform(-1, 1, (m, n))
    outs = []
    for mode in ("1", "0"):
        os.environ["CASC_SPLIT_MODE"] = mode
        try:
            C_hi, C_lo = T(C0), T(np.zeros((m, n)))
            casc.casc_gemm_fp64x2_ex("N", "N", al, *args, be, C_hi, C_lo)
            outs.append((N(C_hi), N(C_lo)))
        finally:
            del os.environ["CASC_SPLIT_MODE"]
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])


# ------------------------------------------------------------------ SYRK (NEXT-4)
@pytest.mark.parametrize("uplo,trans,n,k", [("L", "N", 200, 300), ("U", "N", 129, 513),
                                            ("L", "T", 100, 700), ("U", "T", 65, 256),
                                            ("L", "N", 1100, 600)])
def test_syrk_bitwise_gemm_triangle(casc, orc, uplo, trans, n, k):
    """casc_syrk_fp64x2 runs only the triangle's tiles; every element it stores is
    bitwise the casc_gemm_fp64x2_ex(trans, !trans, A, A) element (same kernel
    arithmetic), the other triangle keeps its NaN sentinel, flags equal the
    oracle's on the triangle, and the triangle is within the north-star bound
    of the exact op(A) op(A)^T."""
    import torch
    d = I.make_config(2, m=n, n=k, k=k, seed=71)
    A_hi, A_lo = d["A_hi"][:n, :k], d["A_lo"][:n, :k]
    Ast = (A_hi.T.copy(), A_lo.T.copy()) if trans == "T" else (A_hi.copy(), A_lo.copy())
    tb = "N" if trans == "T" else "T"
    G_hi = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    G_lo = torch.zeros((n, n), dtype=torch.float64, device="cuda")
    casc.casc_gemm_fp64x2_ex(trans, tb, 1.0, T(Ast[0]), T(Ast[1]), T(Ast[0]), T(Ast[1]), 0.0,
                             G_hi, G_lo)
    S_hi = torch.full((n, n), float("nan"), dtype=torch.float64, device="cuda")
    S_lo = torch.full((n, n), float("nan"), dtype=torch.float64, device="cuda")
    fl = torch.full((n, n), 9, dtype=torch.uint8, device="cuda")
    casc.casc_syrk_fp64x2(uplo, trans, 1.0, T(Ast[0]), T(Ast[1]), 0.0, S_hi, S_lo, flags=fl)
    tri = np.tril(np.ones((n, n), bool)) if uplo == "L" else np.triu(np.ones((n, n), bool))
    s_hi, s_lo, f = N(S_hi), N(S_lo), N(fl)
    assert same_values(s_hi[tri], N(G_hi)[tri]) and same_values(s_lo[tri], N(G_lo)[tri])
    assert np.all(np.isnan(s_hi[~tri])) and np.all(np.isnan(s_lo[~tri])) and np.all(f[~tri] == 9)
    if n <= 200:
        _, _, ofl = orc.casc_syrk(uplo, trans, (1.0, 0.0), *Ast, (0.0, 0.0), np.zeros((n, n)),
                                  np.zeros((n, n)))
        assert np.array_equal(f[tri], ofl[tri])
        ii, jj = np.nonzero(tri)
        r = orc.exact_entries(A_hi, A_lo, A_hi.T.copy(), A_lo.T.copy(), ii, jj, s_hi, s_lo)
        assert np.all(np.abs(r["err"]) <= orc.north_star_bound(k, r["absab"]))


def test_syrk_alpha_beta_and_degenerate(casc, orc):
    """alpha / beta on the triangle (bitwise the GEMM update of the same
    product), k = 0 and alpha = 0 scale only the triangle, bad uplo rejected."""
    import torch
    n, k = 150, 400
    d = I.make_config(1, m=n, n=k, k=k, seed=73)
    A_hi, A_lo = d["A_hi"][:n, :k].copy(), d["A_lo"][:n, :k].copy()
    C0 = np.random.default_rng(2).uniform(-1, 1, (n, n))
    al, be = (1.0 / 3.0, 2.0 ** -56), (-0.7, 2.0 ** -60)
    G_hi, G_lo = T(C0), T(np.zeros((n, n)))
    casc.casc_gemm_fp64x2_ex("N", "T", al, T(A_hi), T(A_lo), T(A_hi), T(A_lo), be, G_hi, G_lo)
    S_hi, S_lo = T(C0), T(np.zeros((n, n)))
    casc.casc_syrk_fp64x2("L", "N", al, T(A_hi), T(A_lo), be, S_hi, S_lo)
    tri = np.tril(np.ones((n, n), bool))
    assert same_values(N(S_hi)[tri], N(G_hi)[tri]) and same_values(N(S_lo)[tri], N(G_lo)[tri])
    assert np.array_equal(N(S_hi)[~tri], C0[~tri])
    # alpha == 0 (and k == 0): C := beta C on the triangle only
    Z_hi, Z_lo = T(C0), T(np.zeros((n, n)))
    casc.casc_syrk_fp64x2("U", "N", 0.0, None, None, (0.5, 0.0), Z_hi, Z_lo)
    up = np.triu(np.ones((n, n), bool))
    assert np.array_equal(N(Z_hi)[up], 0.5 * C0[up]) and np.array_equal(N(Z_hi)[~up], C0[~up])
    with pytest.raises(ValueError):
        casc.casc_syrk_fp64x2("X", "N", 1.0, T(A_hi), T(A_lo), 0.0, S_hi, S_lo)


def test_cuda_graph_capture_replay(casc):
    """The C-ABI calls are stream-ordered with no host synchronisation inside
    (caller workspaces; split modes allocate stream-ordered), so a step can be
    captured into a CUDA graph (torch.cuda.graph) and replayed: bitwise the
    eager results for both cascades, incl. the FP64 cooperative launch (> 148
    tiles) and the INT8 split mode."""
    import torch
    outs = {}
    for n, k in ((832, 300), (1024, 1024)):
        d = I.make_config(1, m=n, n=n, k=k, seed=91)
        A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
        C = [torch.empty(n, n, dtype=torch.float64, device="cuda") for _ in range(4)]
        fl = [torch.empty(n, n, dtype=torch.uint8, device="cuda") for _ in range(2)]
        ws = torch.empty(casc.casc_workspace_bytes(n, n, k), dtype=torch.uint8, device="cuda")
        ws8 = torch.empty(casc.casc_i8_workspace_bytes(n, n, k, 14), dtype=torch.uint8,
                          device="cuda")

        def step():
            casc.casc_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[0], C_lo=C[1], flags=fl[0],
                                  workspace=ws)
            casc.casc_i8_gemm_fp64x2(A_hi, A_lo, B_hi, B_lo, C_hi=C[2], C_lo=C[3], flags=fl[1],
                                     workspace=ws8)

        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        ref = [N(t).copy() for t in C + fl]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for t in C:
            t.fill_(float("nan"))
        g.replay()
        g.replay()
        torch.cuda.synchronize()
        got = [N(t) for t in C + fl]
        outs[n] = all(np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                                     np.ascontiguousarray(b).view(np.uint8))
                      for a, b in zip(got, ref))
    assert all(outs.values()), outs


# ------------------------------------------------------------------ TRSM (NEXT-4)
def _tri_dd(m, uplo, seed, unit=False):
    rng = np.random.default_rng(seed)
    hi = rng.uniform(-1, 1, (m, m)) / m
    hi = np.tril(hi) if uplo == "L" else np.triu(hi)
    lo = hi * 2.0 ** -53 * rng.uniform(-1, 1, (m, m))
    d = 1.0 + rng.uniform(0, 1, m)
    hi[np.arange(m), np.arange(m)] = 1.0 if unit else d
    lo[np.arange(m), np.arange(m)] = 0.0 if unit else d * 2.0 ** -54
    return hi, lo


@pytest.mark.parametrize("uplo,diag,m", [("L", "N", 300), ("U", "N", 600), ("L", "U", 256),
                                         ("U", "U", 70)])
def test_trsm_diag_inverse_bitwise(casc, orc, uplo, diag, m):
    """The TRSM's diagonal-block inverses (FP64x2 substitution, reading R27) are
    bitwise the oracle's, ragged last block and zero fill included."""
    A_hi, A_lo = _tri_dd(m, uplo, 11, diag == "U")
    if diag == "U":  # the diagonal must not be read
        A_hi[np.arange(m), np.arange(m)] = np.nan
    g_hi, g_lo = (N(x) for x in casc.casc_trsm_diag_inv(uplo, diag, T(A_hi), T(A_lo)))
    o_hi, o_lo = orc.trsm_diag_inv(uplo, diag, A_hi, A_lo)
    assert np.array_equal(g_hi.view(np.uint64), o_hi.view(np.uint64))
    assert np.array_equal(g_lo.view(np.uint64), o_lo.view(np.uint64))


@pytest.mark.parametrize("uplo,diag,m,n,trans", [("L", "N", 300, 70, "N"), ("U", "N", 600, 130, "N"),
                                                 ("L", "U", 520, 33, "N"), ("U", "N", 200, 1, "N"),
                                                 ("L", "N", 600, 40, "T"), ("U", "U", 300, 9, "T"),
                                                 ("L", "N", 1100, 20, "N"), ("U", "N", 1300, 7, "T")])
def test_trsm_vs_oracle_and_residual(casc, orc, uplo, diag, m, n, trans):
    """GPU TRSM vs the oracle's (same blocked algorithm; the GEMM updates agree to
    the cascade's bound, not bitwise): within 2^-96 relative on diagonally
    dominant systems, and the residual op(A) X - B small against |A||X|;
    alpha = 2^p scales exactly; strided B untouched outside its columns."""
    import torch
    A_hi, A_lo = _tri_dd(m, uplo, 13, diag == "U")
    rng = np.random.default_rng(15)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))  # normalised pairs: exact scaling
    Xh, Xl = T(B_hi), T(B_lo)
    casc.casc_trsm_fp64x2(uplo, diag, 1.0, T(A_hi), T(A_lo), Xh, Xl, trans=trans)
    x_hi, x_lo = N(Xh), N(Xl)
    o_hi, o_lo = orc.casc_trsm(uplo, diag, (1.0, 0.0), A_hi, A_lo, B_hi, B_lo, trans=trans)
    diff = np.abs((x_hi - o_hi) + (x_lo - o_lo))
    assert np.all(diff <= 2.0 ** -96 * (np.abs(o_hi) + 1e-300) + 2.0 ** -110)
    # residual through the exact evaluator (A X, rows sampled)
    rows = np.unique(np.linspace(0, m - 1, 5).astype(int))
    A_use = A_hi.copy()
    if diag == "U":
        A_use[np.arange(m), np.arange(m)] = 1.0
    opA = (A_use.T.copy(), A_lo.T.copy()) if trans == "T" else (A_use, A_lo)
    ii, jj = np.meshgrid(rows, np.arange(n), indexing="ij")
    r = orc.exact_entries(opA[0], opA[1], x_hi, x_lo, ii.ravel(), jj.ravel(), B_hi, B_lo)
    assert np.all(np.abs(r["err"]) <= 2.0 ** -96 * r["absab"] + 2.0 ** -120)
    # alpha = 4: exact scaling; B as a column window of a wider buffer
    wide_h = T(np.pad(B_hi, ((0, 0), (0, 3)), constant_values=5.0))
    wide_l = T(np.pad(B_lo, ((0, 0), (0, 3)), constant_values=5.0))
    casc.casc_trsm_fp64x2(uplo, diag, 4.0, T(A_hi), T(A_lo), wide_h[:, :n], wide_l[:, :n],
                          trans=trans)
    assert np.array_equal(N(wide_h)[:, :n], 4 * x_hi) and np.array_equal(N(wide_l)[:, :n], 4 * x_lo)
    assert np.all(N(wide_h)[:, n:] == 5.0)


@pytest.mark.parametrize("m,n", [(1, 1), (256, 1), (257, 3), (512, 2)])
def test_trsm_edges(casc, orc, m, n):
    """TRSM at block edges (1 x 1, exactly one block, one row past a block, two
    full blocks), alpha = 0 (X = 0, A never read) and bad arguments."""
    import torch
    A_hi, A_lo = _tri_dd(m, "L", 19)
    rng = np.random.default_rng(23)
    B_hi = rng.uniform(-1, 1, (m, n))
    B_lo = B_hi * 2.0 ** -54 * rng.uniform(-1, 1, (m, n))
    Xh, Xl = T(B_hi), T(B_lo)
    casc.casc_trsm_fp64x2("L", "N", 1.0, T(A_hi), T(A_lo), Xh, Xl)
    o_hi, o_lo = orc.casc_trsm("L", "N", (1.0, 0.0), A_hi, A_lo, B_hi, B_lo)
    diff = np.abs((N(Xh) - o_hi) + (N(Xl) - o_lo))
    assert np.all(diff <= 2.0 ** -96 * np.abs(o_hi) + 2.0 ** -110)
    nanA = T(np.full((m, m), np.nan))
    Zh, Zl = T(B_hi), T(B_lo)
    casc.casc_trsm_fp64x2("U", "U", 0.0, nanA, nanA, Zh, Zl)
    assert np.all(N(Zh) == 0) and np.all(N(Zl) == 0)
    with pytest.raises(ValueError):
        casc.casc_trsm_fp64x2("X", "N", 1.0, T(A_hi), T(A_lo), Xh, Xl)
    with pytest.raises(casc.CascError):  # B overlapping A
        buf_h = torch.zeros((m + 1, m), dtype=torch.float64, device="cuda")
        casc.casc_trsm_fp64x2("L", "N", 1.0, buf_h[:m], buf_h[:m], buf_h[1:, :1], buf_h[1:, :1])


# ------------------------------------------------------------------ column blocks (multi-GPU overlap)
@pytest.mark.parametrize("kind,m,n,k,c0,c1", [("f64", 130, 700, 600, 128, 448),
                                              ("f64", 64, 300, 256, 256, 300),
                                              ("i8", 300, 900, 700, 256, 768),
                                              ("i8", 256, 600, 300, 512, 600)])
def test_packed_column_block_bitwise(casc, kind, m, n, k, c0, c1):
    """casc_gemm_packed_ld / casc_i8_gemm_packed_ld on a column block [c0, c1)
    (packed B offset by whole blocks, C and flags strided views of the full
    arrays): bitwise the same block of the full product, nothing else written
    (the multi-GPU layer multiplies its own slab first, multigpu.py)."""
    import torch
    d = I.make_config(2, m=m, n=n, k=k, seed=97)
    A_hi, A_lo, B_hi, B_lo = (T(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo"))
    if kind == "f64":
        pa, pb = casc.casc_pack_a(A_hi, A_lo), casc.casc_pack_b(B_hi, B_lo)
        blk, W = casc.casc_packed_b_block_bytes(k), 64
        gemm = casc.casc_gemm_packed
    else:
        y = 14
        pa, pb = casc.casc_i8_pack(A_hi, A_lo, False, y), casc.casc_i8_pack(B_hi, B_lo, True, y)
        blk, W = 2 * casc.casc_i8_packed_block_bytes(k, y), 256
        gemm = lambda *a, **kw: casc.casc_i8_gemm_packed(*a, y=y, **kw)
    full = [N(x) for x in gemm(m, n, k, pa, pb)]
    C_hi = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    C_lo = torch.full((m, n), float("nan"), dtype=torch.float64, device="cuda")
    fl = torch.full((m, n), 7, dtype=torch.uint8, device="cuda")
    gemm(m, c1 - c0, k, pa, pb[(c0 // W) * blk:], C_hi=C_hi[:, c0:c1], C_lo=C_lo[:, c0:c1],
         flags=fl[:, c0:c1])
    g = [N(C_hi), N(C_lo), N(fl)]
    for a, b in zip(g, full):
        assert np.array_equal(np.ascontiguousarray(a[:, c0:c1]).view(np.uint8),
                              np.ascontiguousarray(b[:, c0:c1]).view(np.uint8))
    assert np.all(np.isnan(g[0][:, :c0])) and np.all(np.isnan(g[0][:, c1:]))
    assert np.all(g[2][:, :c0] == 7) and np.all(g[2][:, c1:] == 7)


# ------------------------------------------------------------------ full sizes, every entry / cfg3b
def test_cfg1_all_entries_exact(casc, orc):
    """cfg1 (1024^3) at full size through casc_gemm_fp64x2 (small-problem split
    mode, the launch configuration bench.py's small-problem line times): EVERY
    one of the 10^6 entries against the exact product (oracle/exact_fixed.py,
    pinned to the superaccumulator) within the north-star bound, and every flag
    equal to ORACLE-CASCADE's ("all 1M entries checked exactly")."""
    from oracle import exact_fixed as EF
    d = I.make_config(1)
    C_hi, C_lo, flags = run(casc, d)
    err, _ = EF.errors(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], C_hi, C_lo)
    absab = (np.abs(d["A_hi"]) + np.abs(d["A_lo"])) @ (np.abs(d["B_hi"]) + np.abs(d["B_lo"]))
    bound = orc.north_star_bound(1024, absab * (1 - 2.0 ** -40))  # |A||B| to ~1e-13
    assert np.all(np.abs(err) <= bound)
    _, _, o_fl = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    assert np.array_equal(flags, o_fl) and flags.sum() == 0


@pytest.mark.parametrize("variant", ["b", "c"])
def test_cfg3bc_full_size(casc, orc, variant):
    """cfg3 variants b (in-panel pairing) and c (cross-panel pairing), reading
    R13, at FULL size 4096 x 4096 x 32768 on the FP64 path: b flags every entry
    (bin 0 cancels in every panel), c none (the detector is blind across
    panels); flags equal the oracle's on sampled rows, and sampled
    entries stay within eq:cascerr of the exact product (the north-star bound is
    not the bound for adversarial cancellation, reading R14; the flag is)."""
    import torch
    d = I.make_config(3, variant=variant)
    m, n, k = d["m"], d["n"], d["k"]
    C_hi, C_lo, flags = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]),
                                              T(d["B_lo"]))
    torch.cuda.synchronize()
    C_hi, C_lo, flags = N(C_hi), N(C_lo), N(flags)
    assert flags.all() if variant == "b" else not flags.any()
    rows = [0, 2049]
    o_hi, o_lo, o_fl = _sub_oracle(orc, d, rows, n - 64, n)
    assert np.array_equal(flags[rows, n - 64:], o_fl)
    rng = np.random.default_rng(33)
    ii = np.concatenate([rng.integers(0, m, 40), [m - 1]])
    jj = np.concatenate([rng.integers(0, n, 40), [n - 1]])
    r = orc.exact_entries(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"], ii, jj, C_hi, C_lo)
    c = orc.select_widths(k)
    bound = np.zeros(ii.size)
    for p0 in range(0, k, 256):
        a = np.abs(d["A_hi"][ii, p0:p0 + 256])
        b = np.abs(d["B_hi"][p0:p0 + 256, jj])
        absab = np.einsum("tk,kt->t", a, b) * (1 + 2.0 ** -40)
        bound += 2 * orc.cascerr_bound(256, absab, a.max(1), b.max(0), c) \
            + (2 * 128 + 2) * 2.0 ** -104 * absab
    assert np.all(np.abs(r["err"]) <= bound)
