"""The multi-GPU layer's NCCL collective on the GPU (one rank: the only NCCL
world a one-GPU box can form; more ranks on one GPU would be ranks whose
kernels wait on one another, which B200_PROFILING.md rules out).  It runs the
exact call ShardedCascGemm makes -- an asynchronous, in-place
all_gather_into_tensor of a chunk of the packed-B buffer, waited on by the
compute stream -- through NCCL, and the sharded GEMM around it."""

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


def _rank(port, q):
    import torch
    import torch.distributed as dist

    import paper_2303_04353_b200 as casc
    from paper_2303_04353_b200.multigpu import ShardedCascGemm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        out = {"backend": dist.get_backend()}
        m, n, k = 200, 300, 520
        op = ShardedCascGemm(m, n, k, device=torch.device("cuda", 0), gather="packed")
        d = I.make_config(1, m=m, n=n, k=k, seed=5)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        op.own.fill_(7)
        # the production exchange call: asynchronous, in place, waited on by the stream
        work = op._all_gather(op.packed_b_full, op.own, async_op=True)
        work.wait()
        torch.cuda.synchronize()
        out["allgather_ok"] = bool(torch.all(op.packed_b_full == 7).item())
        C = op(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]))
        ref = casc.casc_gemm_fp64x2(T(d["A_hi"]), T(d["A_lo"]), T(d["B_hi"]), T(d["B_lo"]))
        torch.cuda.synchronize()
        out["bitwise"] = all(torch.equal(a.view(torch.uint8) if a.dtype != torch.uint8 else a,
                                         b.view(torch.uint8) if b.dtype != torch.uint8 else b)
                             for a, b in zip(C, ref))
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_nccl_exchange_call_one_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_rank, args=(_free_port(), q))
    p.start()
    out = q.get(timeout=240)
    p.join(timeout=60)
    assert p.exitcode == 0
    assert out == {"backend": "nccl", "allgather_ok": True, "bitwise": True}
