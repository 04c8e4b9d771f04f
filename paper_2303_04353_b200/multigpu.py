"""Multi-GPU layer: C row-block sharded over ranks, B's packed slices exchanged
once over NVLink (BASELINE north star: "partitions C into row/column blocks
across the 8xB200 box, with B (or A) slices broadcast over NVLink through
NCCL").

One process per GPU (torch.distributed, NCCL).  Rank r of W:
  1. packs its rows [r0, r1) of A (casc_pack_a; per-row scales are row-local);
  2. packs its column slab of B (casc_pack_b; per-column scales are
     column-local, so the slab's packed bytes are bit-identical to the same
     blocks of a single-GPU pack);
  3. all-gathers the packed B slabs (one ncclAllGather of equal-size chunks;
     the packed layout is 64-column-block major, so the gathered buffer IS
     the packed B of the whole matrix);
  4. runs the fused cascaded GEMM on its rows (casc_gemm_packed).
k is never split, so there is no reduction and every element is computed by
exactly the same arithmetic as on one GPU: C is bitwise independent of W
(P-invariance).

The INT8 cascade (NEXT-3) shards the same way: its packed B is also
column-block major (128-column blocks, counted in pairs), so a 256-multiple
slab is a byte range of the full packed B (`i8_cuda_ops`, block = 256).

`ops` makes the kernels injectable so the host-side plumbing (sharding,
padding, gather order) is testable on CPU with the gloo backend.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

BLOCK = 64  # packed column-block width of the FP64 cascade (casc_layout.cuh TN)
I8_BLOCK = 256  # slab granularity of the INT8 cascade (two 128-column packed blocks)


def row_shard(m: int, world: int, rank: int):
    """Rows [r0, r1) of A and C owned by `rank` (balanced, contiguous)."""
    return (rank * m) // world, ((rank + 1) * m) // world


def col_slab(n: int, world: int, rank: int, block: int = BLOCK):
    """Columns [c0, c1) of B packed by `rank`: equal block-multiple slabs so
    every rank contributes the same number of packed blocks to the all-gather."""
    nb = -(-n // block)
    per = -(-nb // world)
    c0 = min(n, rank * per * block)
    c1 = min(n, (rank + 1) * per * block)
    return c0, c1, per


@dataclass
class Ops:
    pack_a: object
    pack_b: object
    gemm_packed: object
    packed_b_block_bytes: object
    launch_count: object = None  # launches of the last call (our kernels)


def cuda_ops() -> Ops:
    import paper_2303_04353_b200 as casc
    return Ops(pack_a=casc.casc_pack_a, pack_b=casc.casc_pack_b,
               gemm_packed=casc.casc_gemm_packed,
               packed_b_block_bytes=casc.casc_packed_b_block_bytes,
               launch_count=casc.casc_last_launch_count)


def i8_cuda_ops(y: int = 14) -> Ops:
    """The INT8 cascade's entry points with the Ops contracts (block = 256 columns)."""
    import paper_2303_04353_b200 as casc

    def pack_a(A_hi, A_lo, packed=None):
        return casc.casc_i8_pack(A_hi, A_lo, False, y, packed=packed)

    def pack_b(B_hi, B_lo, packed):
        return casc.casc_i8_pack(B_hi, B_lo, True, y, packed=packed)

    def gemm_packed(m, n, k, pa, pb, C_hi=None, C_lo=None, flags=None):
        return casc.casc_i8_gemm_packed(m, n, k, pa, pb, y, C_hi=C_hi, C_lo=C_lo, flags=flags)

    return Ops(pack_a=pack_a, pack_b=pack_b, gemm_packed=gemm_packed,
               packed_b_block_bytes=lambda k: 2 * casc.casc_i8_packed_block_bytes(k, y),
               launch_count=casc.casc_last_launch_count)


class ShardedCascGemm:
    """Row-sharded cascaded FP64x2 GEMM for one (m, n, k) problem.  Buffers are
    allocated once and reused across calls (bench steps)."""

    def __init__(self, m: int, n: int, k: int, group=None, ops: Ops | None = None,
                 device=None, block: int = BLOCK, gather: str = "packed"):
        """block: slab granularity (columns) of the packed B: 64 for the FP64
        cascade, I8_BLOCK with i8_cuda_ops().
        gather: what the ranks exchange (N > 1).  "packed": each rank splits its
        column slab of B and the packed slabs are all-gathered (FP64 cascade:
        56 B per element of B; INT8 cascade: ~14 B).  "raw": the FP64x2 slabs
        themselves are all-gathered (16 B per element) and every rank splits all
        of B locally, slab by slab into the packed layout (the byte-cheaper
        choice for the FP64 cascade).  Bitwise the same result."""
        if gather not in ("packed", "raw"):
            raise ValueError("gather must be 'packed' or 'raw'")
        self.m, self.n, self.k = m, n, k
        self.block = block
        self.gather = gather
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.ops = ops or cuda_ops()
        self.device = device if device is not None else torch.device("cuda")
        self.r0, self.r1 = row_shard(m, self.world, self.rank)
        self.c0, self.c1, self.blocks_per_rank = col_slab(n, self.world, self.rank, block)
        blk = self.ops.packed_b_block_bytes(k)
        self.chunk = self.blocks_per_rank * blk
        self.packed_b_local = torch.zeros(self.chunk, dtype=torch.uint8, device=self.device)
        self.packed_b_full = (torch.empty(self.chunk * self.world, dtype=torch.uint8,
                                          device=self.device) if self.world > 1 else None)
        self.packed_a = None
        self.raw = self.gather == "raw" and self.world > 1
        if self.raw:  # [rank][hi | lo][k][slab width padded to whole blocks]
            self.wpad = self.blocks_per_rank * block
            self.raw_local = torch.zeros((2, k, self.wpad), dtype=torch.float64,
                                         device=self.device)
            self.raw_full = torch.empty((self.world, 2, k, self.wpad), dtype=torch.float64,
                                        device=self.device)
            self.slabs = [col_slab(n, self.world, r, block)[:2] for r in range(self.world)]
        # names of the intervals between the 4 events of __call__ (bench phases)
        self.phase_names = (["split_a", "allgather_raw", "split_b", "gemm"] if self.raw else
                            ["split_a", "split_b", "allgather", "gemm"])

    def __call__(self, A_hi_rows, A_lo_rows, B_hi_slab, B_lo_slab, C_hi=None, C_lo=None,
                 flags=None, events=None):
        """A_*_rows: this rank's rows (r1-r0) x k.  B_*_slab: k x (c1-c0).
        Returns this rank's (C_hi, C_lo, flags) rows.  `events`, if given, is a
        list of 4 CUDA events recorded after pack_a, pack_b, all-gather, gemm."""
        mloc = self.r1 - self.r0
        count = getattr(self.ops, "launch_count", None) or (lambda: 0)
        self.launches = 0
        self.packed_a = self.ops.pack_a(A_hi_rows, A_lo_rows, packed=self.packed_a)
        self.launches += count()
        rec = (lambda i: events[i].record()) if events else (lambda i: None)
        rec(0)
        if self.raw:
            w = self.c1 - self.c0
            if w > 0:
                self.raw_local[0, :, :w].copy_(B_hi_slab)
                self.raw_local[1, :, :w].copy_(B_lo_slab)
            if dist.get_backend(self.group) == "gloo":  # CPU plumbing tests
                dist.all_gather(list(self.raw_full.unbind(0)), self.raw_local, group=self.group)
            else:  # NCCL over NVLink / NVSwitch
                dist.all_gather_into_tensor(self.raw_full.view(-1), self.raw_local.view(-1),
                                            group=self.group)
            rec(1)
            blk = self.ops.packed_b_block_bytes(self.k)
            for r, (a0, a1) in enumerate(self.slabs):
                if a1 > a0:
                    used = -(-(a1 - a0) // self.block) * blk
                    base = r * self.chunk
                    self.ops.pack_b(self.raw_full[r, 0, :, :a1 - a0],
                                    self.raw_full[r, 1, :, :a1 - a0],
                                    packed=self.packed_b_full[base:base + used])
                    self.launches += count()
            rec(2)
            out = self.ops.gemm_packed(mloc, self.n, self.k, self.packed_a, self.packed_b_full,
                                       C_hi=C_hi, C_lo=C_lo, flags=flags)
            self.launches += count()
            rec(3)
            return out
        if self.c1 > self.c0:
            used = -(-(self.c1 - self.c0) // self.block) * self.ops.packed_b_block_bytes(self.k)
            self.ops.pack_b(B_hi_slab, B_lo_slab, packed=self.packed_b_local[:used])
            self.launches += count()
        rec(1)
        if self.world > 1:
            if dist.get_backend(self.group) == "gloo":  # CPU plumbing tests
                dist.all_gather(list(self.packed_b_full.chunk(self.world)), self.packed_b_local,
                                group=self.group)
            else:  # NCCL over NVLink / NVSwitch
                dist.all_gather_into_tensor(self.packed_b_full, self.packed_b_local,
                                            group=self.group)
            pb = self.packed_b_full
        else:
            pb = self.packed_b_local
        rec(2)
        out = self.ops.gemm_packed(mloc, self.n, self.k, self.packed_a, pb, C_hi=C_hi,
                                   C_lo=C_lo, flags=flags)
        self.launches += count()
        rec(3)
        return out
