"""Multi-GPU host logic on CPU (-m "not gpu"): world_size 2 with the gloo
backend.  The CUDA kernels are replaced by CPU stand-ins built on the oracle
(tests may call the oracle); what is under test is the product's plumbing in
paper_2303_04353_b200/multigpu.py: row sharding, 64-column slab assignment
with padding, the all-gather of packed slabs, and P-invariance of C."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import casc_inputs as I


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_arithmetic():
    from paper_2303_04353_b200.multigpu import col_slab, row_shard
    for m in (1, 7, 64, 1000, 16384):
        for w in (1, 2, 3, 4, 8):
            rows = [row_shard(m, w, r) for r in range(w)]
            assert rows[0][0] == 0 and rows[-1][1] == m
            assert all(rows[i][1] == rows[i + 1][0] for i in range(w - 1))
    for n in (1, 63, 64, 150, 1000, 16384):
        for w in (1, 2, 4, 8):
            slabs = [col_slab(n, w, r) for r in range(w)]
            assert slabs[0][0] == 0 and slabs[-1][1] == n
            per = slabs[0][2]
            assert all(s[2] == per for s in slabs) and per * w * 64 >= n
            for c0, c1, _ in slabs:
                assert c1 == c0 or (c0 % 64 == 0 and c1 - c0 <= per * 64)


class _CpuOps:
    """CPU stand-ins with the same contracts as the CUDA entry points: packed B
    is column-block major (each block = raw hi | lo of k x W, zero-padded; W =
    64 for the FP64 cascade, 256 for the INT8 cascade's slab unit), and the
    product is the matching oracle."""

    def __init__(self, k, W=64, i8=False):
        self.k = k
        self.W = W
        self.i8 = i8

    def packed_b_block_bytes(self, k):
        return 2 * k * self.W * 8

    def pack_a(self, A_hi, A_lo, packed=None):
        return (A_hi.clone(), A_lo.clone())

    def pack_b(self, B_hi, B_lo, packed):
        k, w = B_hi.shape
        W = self.W
        nb = -(-w // W)
        buf = packed.view(torch.float64).view(nb, 2, k, W)
        buf.zero_()
        for j in range(nb):
            c = B_hi[:, W * j:W * (j + 1)]
            buf[j, 0, :, :c.shape[1]] = c
            buf[j, 1, :, :c.shape[1]] = B_lo[:, W * j:W * (j + 1)]
        return packed

    def gemm_packed(self, m, n, k, pa, pb, C_hi=None, C_lo=None, flags=None):
        import oracle
        W = self.W
        nb = -(-n // W)
        blocks = pb.view(torch.float64)[:nb * 2 * k * W].view(nb, 2, k, W)
        B_hi = torch.cat([blocks[j, 0] for j in range(nb)], dim=1)[:, :n].numpy()
        B_lo = torch.cat([blocks[j, 1] for j in range(nb)], dim=1)[:, :n].numpy()
        fn = oracle.i8_casc_gemm if self.i8 else oracle.casc_gemm
        h, l, f = fn(pa[0].numpy(), pa[1].numpy(), B_hi, B_lo)
        out = []
        for dst, src in ((C_hi, h), (C_lo, l), (flags, f)):  # C may be a column block
            if dst is None:
                dst = torch.from_numpy(src)
            else:
                dst.copy_(torch.from_numpy(src))
            out.append(dst)
        return tuple(out)


def _worker(rank, world, port, m, n, k, out, i8=False, gather="packed", overlap=True):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2303_04353_b200.multigpu import I8_BLOCK, ShardedCascGemm
    W = I8_BLOCK if i8 else 64
    op = ShardedCascGemm(m, n, k, ops=_CpuOps(k, W, i8), device=torch.device("cpu"), block=W,
                         gather=gather, overlap=overlap)
    d = I.make_config(1, m=m, n=n, k=k, seed=21, rows=slice(op.r0, op.r1))
    A_hi, A_lo = torch.from_numpy(d["A_hi"]), torch.from_numpy(d["A_lo"])
    B_hi = torch.from_numpy(d["B_hi"][:, op.c0:op.c1].copy())
    B_lo = torch.from_numpy(d["B_lo"][:, op.c0:op.c1].copy())
    C_hi, C_lo, fl = op(A_hi, A_lo, B_hi, B_lo)
    np.savez(os.path.join(out, f"r{rank}.npz"), C_hi=C_hi.numpy(), C_lo=C_lo.numpy(),
             fl=fl.numpy(), r0=op.r0, r1=op.r1, gather=op.gather)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,m,n,k,gather,overlap", [
    (2, 10, 150, 300, "packed", True), (2, 7, 64, 40, "packed", True),
    (2, 10, 150, 300, "raw", True), (2, 5, 200, 70, "raw", True),
    (2, 10, 150, 300, "packed", False), (2, 5, 200, 70, "raw", False),
    (4, 9, 300, 80, "packed", True), (4, 6, 200, 70, "raw", True), (4, 9, 130, 40, "packed", False),
    (2, 10, 150, 300, "p2p", True), (4, 6, 200, 70, "p2p", True)])
def test_gloo_world_p_invariance(tmp_path, orc, world, m, n, k, gather, overlap):
    """The production exchange (in-place all_gather_into_tensor, the call NCCL
    runs on the GPUs) on gloo: world 2 and 4, packed and raw exchanges, with
    the overlapped schedule (own column slab multiplied while the exchange
    runs, then the other columns) and the serial one: the same bits as one
    process.  gather="raw" exchanges the FP64x2 slabs and packs all of B on
    every rank (SURVEY §8(e) byte-cheaper alternative).  gather="p2p" needs
    CUDA IPC: here no rank can export a device buffer, so every rank falls back
    together (collective decision) to the raw all-gather: the same bits."""
    mp.spawn(_worker, args=(world, _free_port(), m, n, k, str(tmp_path), False, gather, overlap),
             nprocs=world, join=True)
    d = I.make_config(1, m=m, n=n, k=k, seed=21)
    ref_hi, ref_lo, ref_fl = orc.casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    rows = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        r0, r1 = int(z["r0"]), int(z["r1"])
        assert np.array_equal(z["C_hi"], ref_hi[r0:r1])
        assert np.array_equal(z["C_lo"], ref_lo[r0:r1])
        assert np.array_equal(z["fl"], ref_fl[r0:r1])
        assert str(z["gather"]) == ("raw" if gather == "p2p" else gather)
        rows += r1 - r0
    assert rows == m


@pytest.mark.parametrize("world,m,n,k", [(2, 9, 600, 70), (2, 4, 256, 33), (4, 8, 900, 40)])
def test_gloo_world_i8_p_invariance(tmp_path, orc, world, m, n, k):
    """The INT8 cascade's sharding (256-column slabs, NEXT-3), overlapped
    exchange: the gathered result equals the single-process oracle bit for bit."""
    mp.spawn(_worker, args=(world, _free_port(), m, n, k, str(tmp_path), True), nprocs=world,
             join=True)
    d = I.make_config(1, m=m, n=n, k=k, seed=21)
    ref_hi, ref_lo, ref_fl = orc.i8_casc_gemm(d["A_hi"], d["A_lo"], d["B_hi"], d["B_lo"])
    rows = 0
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        r0, r1 = int(z["r0"]), int(z["r1"])
        assert np.array_equal(z["C_hi"], ref_hi[r0:r1])
        assert np.array_equal(z["C_lo"], ref_lo[r0:r1])
        assert np.array_equal(z["fl"], ref_fl[r0:r1])
        rows += r1 - r0
    assert rows == m
