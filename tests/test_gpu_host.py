"""casc_gemm_fp64x2_host: operands in host memory, streamed through the GPU in
blocks of row slabs of A x column slabs of B (include/casc.h).  The result must
be bitwise the device-resident casc_gemm_fp64x2 result (blocks change nothing:
an element of C depends only on its row of A and column of B, and the scale
exponents are per row / column), for ragged slab counts in both directions,
pinned and pageable buffers, strided host views and the degenerate cases."""

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


def device_ref(casc, d):
    import torch
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    out = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]))
    return [x.cpu().numpy() for x in out]


def bitwise(x, y):
    return np.array_equal(np.ascontiguousarray(x).view(np.uint64),
                          np.ascontiguousarray(y).view(np.uint64))


@pytest.mark.parametrize("m,n,k,slab,scol,pinned", [
    (300, 257, 700, 64, 64, True), (130, 200, 513, 64, 128, False), (1000, 300, 1100, 0, 0, True),
    (2048, 1024, 1024, 512, 256, True), (65, 64, 9000, 128, 0, True), (1, 1, 1, 0, 0, False),
    (200, 1000, 300, 0, 192, True),
    # m, n >= 8192: the default wave-aligned blocks (4096 x 2368 on 148 SMs), ragged both ways
    (8200, 9000, 300, 0, 0, True)])
def test_host_bitwise_device(casc, m, n, k, slab, scol, pinned):
    import torch
    d = I.make_config(2, m=m, n=n, k=k, seed=51)
    ref = device_ref(casc, d)
    H = lambda a: (torch.from_numpy(np.ascontiguousarray(a)).pin_memory() if pinned
                   else torch.from_numpy(np.ascontiguousarray(a)))
    C_hi, C_lo, fl = casc.casc_gemm_fp64x2_host(H(d["A_hi"]), H(d["A_lo"]), H(d["B_hi"]),
                                                H(d["B_lo"]), slab_rows=slab, slab_cols=scol)
    assert bitwise(C_hi.numpy(), ref[0]) and bitwise(C_lo.numpy(), ref[1])
    assert np.array_equal(fl.numpy(), ref[2])


def test_host_strided_views_no_flags_and_degenerate(casc):
    import torch
    m, n, k = 200, 150, 600
    d = I.make_config(1, m=m, n=n, k=k, seed=53)
    ref = device_ref(casc, d)
    # operands as column windows of wider pinned host buffers (lda > k, ldb > n, ldc > n)
    wide = lambda a, extra: torch.from_numpy(np.pad(a, ((0, 0), (0, extra)))).pin_memory()
    A_hi, A_lo = wide(d["A_hi"], 37), wide(d["A_lo"], 37)
    B_hi, B_lo = wide(d["B_hi"], 11), wide(d["B_lo"], 11)
    C_hi = torch.full((m, n + 9), 7.0, dtype=torch.float64).pin_memory()
    C_lo = torch.full((m, n + 9), 7.0, dtype=torch.float64).pin_memory()
    casc.casc_gemm_fp64x2_host(A_hi[:, :k], A_lo[:, :k], B_hi[:, :n], B_lo[:, :n],
                               C_hi=C_hi[:, :n], C_lo=C_lo[:, :n], want_flags=False,
                               slab_rows=64, slab_cols=64)
    assert bitwise(C_hi[:, :n].numpy(), ref[0]) and bitwise(C_lo[:, :n].numpy(), ref[1])
    assert np.all(C_hi[:, n:].numpy() == 7.0) and np.all(C_lo[:, n:].numpy() == 7.0)
    # k == 0: C := 0, flags := 0
    z = torch.empty((m, 0), dtype=torch.float64)
    zb = torch.empty((0, n), dtype=torch.float64)
    c0, c1, f0 = casc.casc_gemm_fp64x2_host(z, z, zb, zb)
    assert np.all(c0.numpy() == 0) and np.all(c1.numpy() == 0) and np.all(f0.numpy() == 0)
    # bad arguments: negative slab, CUDA tensors where host ones are expected
    h = torch.zeros((4, 4), dtype=torch.float64)
    with pytest.raises(casc.CascError):
        casc.casc_gemm_fp64x2_host(h, h, h, h, slab_rows=-1)
    with pytest.raises(casc.CascError):
        casc.casc_gemm_fp64x2_host(h, h, h, h, slab_cols=-1)
    with pytest.raises(TypeError):
        casc.casc_gemm_fp64x2_host(h.cuda(), h.cuda(), h, h)


def test_host_repeated_calls_reuse_pool(casc):
    """Back-to-back calls on one stream (buffers from the stream-ordered pool,
    internal streams and events reused) stay bitwise stable."""
    import torch
    d = I.make_config(1, m=600, n=400, k=800, seed=57)
    P = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    args = [P(d[x]) for x in ("A_hi", "A_lo", "B_hi", "B_lo")]
    outs = [casc.casc_gemm_fp64x2_host(*args, slab_rows=128, slab_cols=128, sync=False)
            for _ in range(3)]
    torch.cuda.current_stream().synchronize()
    ref = device_ref(casc, d)
    for o in outs:
        assert bitwise(o[0].numpy(), ref[0]) and bitwise(o[1].numpy(), ref[1])
