"""Re-entrancy of the C ABI (include/casc.h conventions): calls
on different CUDA streams and host threads share no device memory and never
synchronise the host, so concurrent calls give bitwise the serial results and
cannot hang (the fused FP64 kernel's tile-wave barrier is per launch and
bounded; its workspace is the caller's or a stream-ordered allocation)."""

import threading

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


def _inputs(seed, m, n, k):
    import torch
    d = I.make_config(1, m=m, n=n, k=k, seed=seed)
    return [torch.from_numpy(d[x]).cuda() for x in ("A_hi", "A_lo", "B_hi", "B_lo")]


def _eq(x, y):
    import torch
    return all(torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                           b.view(torch.uint8) if b.dtype != torch.uint8 else b)
               for a, b in zip(x, y))


# shapes with more 64 x 64 tiles than SMs (the fused kernel's wave barrier is
# active) and k > 256 (several panels)
SHAPES = [(1536, 1280, 768), (1280, 1536, 1024)]


def test_concurrent_streams_bitwise(casc):
    """Both cascades and the library-workspace FP64 entry, interleaved on two
    streams with different inputs, several times over: bitwise the serial
    results, no hang."""
    import torch
    ins = [_inputs(100 + i, *SHAPES[i]) for i in range(2)]
    serial = []
    for i in range(2):
        serial.append((casc.casc_gemm_fp64x2(*ins[i]), casc.casc_i8_gemm_fp64x2(*ins[i])))
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(2)]
    for s in streams:
        s.wait_stream(torch.cuda.current_stream())
    outs = [[], []]
    for rep in range(3):
        for i in range(2):
            with torch.cuda.stream(streams[i]):
                outs[i].append((casc.casc_gemm_fp64x2(*ins[i], stream=streams[i]),
                                casc.casc_i8_gemm_fp64x2(*ins[i], stream=streams[i])))
    torch.cuda.synchronize()
    for i in range(2):
        for f64, i8 in outs[i]:
            assert _eq(f64, serial[i][0]) and _eq(i8, serial[i][1])


def test_concurrent_host_threads_bitwise(casc):
    """Host threads, each with its own stream, calling the FP64 cascade (library
    workspace and caller workspace) at the same time."""
    import torch
    ins = [_inputs(200 + i, 1280, 1280, 640) for i in range(3)]
    ref = [casc.casc_gemm_fp64x2(*x) for x in ins]
    torch.cuda.synchronize()
    results = [None] * 3
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ws = None
                if i == 2:
                    ws = torch.empty(casc.casc_workspace_bytes(1280, 1280, 640), dtype=torch.uint8,
                                     device="cuda")
                r = [casc.casc_gemm_fp64x2(*ins[i], stream=s, workspace=ws) for _ in range(2)]
            s.synchronize()
            results[i] = r
        except Exception as e:  # noqa: BLE001
            errors.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(3)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not errors, errors
    for i in range(3):
        for r in results[i]:
            assert _eq(r, ref[i])


def test_finalize_returns_pool_memory(casc):
    """casc_finalize trims the device pool the per-call workspaces come from;
    calls afterwards still work."""
    import torch
    x = _inputs(300, 512, 512, 512)
    ref = casc.casc_gemm_fp64x2(*x)
    torch.cuda.synchronize()
    casc.casc_finalize()
    casc.casc_i8_finalize()
    again = casc.casc_gemm_fp64x2(*x)
    torch.cuda.synchronize()
    assert _eq(again, ref)
