"""The multi-GPU layer with the REAL CUDA path, two processes on the one GPU
this build has (gloo backend for the exchange; the ranks' kernels never wait
on each other, so sharing a device is safe): every rank runs the production
pack / all-gather / packed-GEMM sequence of ShardedCascGemm on its rows, and
the gathered C is bitwise the single-process result (P-invariance: k is never
split), for the FP64 cascade ('raw' and 'packed' exchanges, and 'p2p': the
slabs pulled from the other process's exported buffer by the copy engine, CUDA
IPC within the one device, called twice to exercise the reuse ordering) and
the INT8 cascade ('packed', 'p2p'); 'p2pfail': one rank cannot map the
other's buffer, so both fall back to the raw all-gather together."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import casc_inputs as I

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, m, n, k, kind, q):
    import torch
    import torch.distributed as dist

    from paper_2303_04353_b200.multigpu import (BLOCK, I8_BLOCK, ShardedCascGemm, col_slab,
                                                i8_cuda_ops, row_shard)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        i8 = kind in ("i8", "i8p2p")
        block = I8_BLOCK if i8 else BLOCK
        r0, r1 = row_shard(m, world, rank)
        c0, c1, _ = col_slab(n, world, rank, block)
        d = I.make_config(1, m=m, n=n, k=k, seed=77)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        gather = {"i8": "packed", "packed": "packed", "raw": "raw", "p2p": "p2p",
                  "i8p2p": "p2p", "p2pfail": "p2p"}[kind]
        if kind == "p2pfail":  # rank 1 cannot map rank 0's buffer: both fall back
            os.environ["CASC_P2P_FAIL_RANK"] = "1"
        op = ShardedCascGemm(m, n, k, ops=i8_cuda_ops() if i8 else None,
                             device=torch.device("cuda", 0), block=block, gather=gather)
        args = (T(d["A_hi"][r0:r1]), T(d["A_lo"][r0:r1]), T(d["B_hi"][:, c0:c1]),
                T(d["B_lo"][:, c0:c1]))
        if kind == "p2pfail":
            assert op.gather == "raw" and not op.p2p
        C_hi, C_lo, fl = op(*args)
        if gather == "p2p":  # a second call reuses the exported buffers (ordering barriers)
            C_hi, C_lo, fl = op(*args)
        torch.cuda.synchronize()
        q.put((rank, C_hi.cpu().numpy(), C_lo.cpu().numpy(), fl.cpu().numpy()))
        op.close()
        dist.barrier()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,m,n,k", [("raw", 300, 520, 700), ("packed", 257, 200, 300),
                                        ("i8", 600, 700, 900), ("p2p", 300, 520, 700),
                                        ("i8p2p", 600, 700, 900), ("p2pfail", 300, 520, 700)])
def test_two_processes_one_gpu_bitwise(kind, m, n, k):
    import torch

    import paper_2303_04353_b200 as casc
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank, args=(r, 2, port, m, n, k, kind, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict((r, (h, l, f)) for r, h, l, f in (q.get(timeout=240) for _ in range(2)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    C = [np.concatenate([got[0][i], got[1][i]]) for i in range(3)]
    d = I.make_config(1, m=m, n=n, k=k, seed=77)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    fn = casc.casc_i8_gemm_fp64x2 if kind in ("i8", "i8p2p") else casc.casc_gemm_fp64x2
    ref = [x.cpu().numpy() for x in fn(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]))]
    for a, b in zip(C, ref):
        assert np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                              np.ascontiguousarray(b).view(np.uint8))
