"""Multi-GPU layer: C row-block sharded over ranks, B's packed slices exchanged
once over NVLink (BASELINE north star: "partitions C into row/column blocks
across the 8xB200 box, with B (or A) slices broadcast over NVLink through
NCCL").

One process per GPU (torch.distributed, NCCL).  Rank r of W:
  1. packs its rows [r0, r1) of A (casc_pack_a; per-row scales are row-local);
  2. packs its column slab of B (casc_pack_b; per-column scales are
     column-local, so the slab's packed bytes are bit-identical to the same
     blocks of a single-GPU pack);
  3. all-gathers the packed B slabs (one in-place ncclAllGather of equal-size
     chunks; the packed layout is 64-column-block major, so the gathered
     buffer IS the packed B of the whole matrix) -- while
  4. the fused cascaded GEMM multiplies its rows by its OWN column slab
     (casc_gemm_packed_ld on that column block of C); once the exchange has
     landed (stream-ordered wait, no kernel spins on another), a second
     launch multiplies the other columns.
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
                 device=None, block: int = BLOCK, gather: str = "packed",
                 overlap: bool = True):
        """block: slab granularity (columns) of the packed B: 64 for the FP64
        cascade, I8_BLOCK with i8_cuda_ops().
        gather: what the ranks exchange (N > 1).  "packed": each rank splits its
        column slab of B and the packed slabs are all-gathered (FP64 cascade:
        56 B per element of B; INT8 cascade: ~14 B).  "raw": the FP64x2 slabs
        themselves are all-gathered (16 B per element) and every rank splits all
        of B locally, slab by slab into the packed layout (the byte-cheaper
        choice for the FP64 cascade).  Bitwise the same result.
        "p2p": no collective; every rank exports the device buffer holding its
        packed slab (CUDA IPC), maps the others' and PULLS their slabs with the
        copy engines (casc_copy_async on two copy streams), so the exchange takes
        no SM from the GEMM and each slab's GEMM starts as soon as that slab has
        landed (own slab first, then r+1, r+2, ...); ordering between ranks is
        two CPU barriers per call (gloo group), no kernel waits on another rank.
        Call close() on every rank when done (it unmaps the peers' buffers and
        frees the exported one; collective).  If any rank cannot export or map
        a buffer, every rank falls back to "raw" (collective decision).
        overlap (N > 1): the exchange runs while the GEMM multiplies the rank's
        own column slab (casc_gemm_packed_ld on a column block of C), then the
        other columns are multiplied once it has landed -- two stream-ordered
        launches, no kernel waits on another (B200_PROFILING.md); bitwise the
        same C, since every element depends only on its row and column."""
        if gather not in ("packed", "raw", "p2p"):
            raise ValueError("gather must be 'packed', 'raw' or 'p2p'")
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
        self.blk = blk
        self.chunk = self.blocks_per_rank * blk
        self.overlap = overlap and self.world > 1
        # packed B of all ranks: chunk r = rank r's column slab (column-block major,
        # so the gathered buffer IS the packed B of the whole matrix); with one
        # rank it is just the local pack
        self.p2p = gather == "p2p" and self.world > 1
        self._ipc_ptr = None
        if self.p2p and not self._setup_p2p():
            # some rank could not export or map a buffer: every rank falls back
            # (decided collectively) to the NCCL all-gather of raw slabs
            self.p2p = False
            self.gather = gather = "raw"
        if not self.p2p:
            self.packed_b_full = torch.zeros(self.chunk * self.world, dtype=torch.uint8,
                                             device=self.device)
        self.own = self.packed_b_full[self.rank * self.chunk:(self.rank + 1) * self.chunk]
        self.packed_a = None
        self.raw = self.gather == "raw" and self.world > 1
        if self.raw:  # [rank][hi | lo][k][slab width padded to whole blocks]
            self.wpad = self.blocks_per_rank * block
            self.raw_full = torch.zeros((self.world, 2, k, self.wpad), dtype=torch.float64,
                                        device=self.device)
        self.slabs = [col_slab(n, self.world, r, block)[:2] for r in range(self.world)]
        # names of the intervals between the 5 events of __call__ (bench phases)
        if self.p2p:
            self.phase_names = ["split_a", "split_b_own", "gemm_own_cols",
                                "gemm_other_cols_p2p"]
        elif self.overlap:
            self.phase_names = ["split_a", "split_b_own", "gemm_own_cols", "gemm_other_cols"]
        elif self.raw:
            self.phase_names = ["split_a", "allgather_raw", "split_b", "gemm"]
        else:
            self.phase_names = ["split_a", "split_b", "allgather", "gemm"]
        self.launches = 0

    def _setup_p2p(self) -> bool:
        """Export this rank's packed-B buffer, map every other rank's (CUDA IPC).
        Collective over a gloo group; returns False on every rank (after undoing
        what was set up) if any rank failed."""
        import paper_2303_04353_b200 as casc
        self._casc = casc
        self.cpu_group = dist.new_group(backend="gloo")
        self.peer_ptrs = {}
        handle, ok = None, True
        try:
            with torch.cuda.device(self.device):
                self._ipc_ptr, handle, self.packed_b_full = casc.casc_ipc_alloc(
                    self.chunk * self.world)
        except Exception:
            ok = False
        handles = [None] * self.world
        dist.all_gather_object(handles, handle if ok else None, group=self.cpu_group)
        ok = ok and all(h is not None for h in handles)
        if ok:
            try:
                import os
                # test hook: this rank fails to map its peers' buffers
                if os.environ.get("CASC_P2P_FAIL_RANK") == str(self.rank):
                    raise RuntimeError("CASC_P2P_FAIL_RANK")
                with torch.cuda.device(self.device):
                    for q in range(self.world):
                        if q != self.rank:
                            self.peer_ptrs[q] = casc.casc_ipc_open(handles[q])
            except Exception:
                ok = False
        oks = [None] * self.world
        dist.all_gather_object(oks, ok, group=self.cpu_group)
        if all(oks):
            with torch.cuda.device(self.device):
                self.copy_streams = [torch.cuda.Stream(self.device) for _ in range(2)]
                self.slab_events = [torch.cuda.Event() for _ in range(self.world)]
                self.copy_done = [torch.cuda.Event() for _ in self.copy_streams]
            self.copies_pending = False
            return True
        for ptr in self.peer_ptrs.values():
            casc.casc_ipc_close(ptr)
        dist.barrier(group=self.cpu_group)  # every mapping closed before the frees
        self.peer_ptrs = {}
        self.packed_b_full = None
        if self._ipc_ptr is not None:
            casc.casc_ipc_free(self._ipc_ptr)
            self._ipc_ptr = None
        return False

    def _all_gather(self, full, mine, async_op=False):
        """In-place all-gather of equal chunks (rank r's chunk at offset r): one
        all_gather_into_tensor for every backend (NCCL over NVLink / NVSwitch on
        the GPUs, gloo in the CPU tests)."""
        return dist.all_gather_into_tensor(full, mine, group=self.group, async_op=async_op)

    def _used(self, a0, a1):
        return -(-(a1 - a0) // self.block) * self.blk

    def _pack_slab(self, r, B_hi, B_lo, count):
        a0, a1 = self.slabs[r]
        if a1 > a0:
            base = r * self.chunk
            self.ops.pack_b(B_hi, B_lo, packed=self.packed_b_full[base:base + self._used(a0, a1)])
            self.launches += count()

    def _gemm_cols(self, pa, col0, col1, C_hi, C_lo, flags, count):
        """C[:, col0:col1] from the packed blocks of those columns (col0 a slab
        boundary: a byte range of the packed B)."""
        if col1 <= col0:
            return
        mloc = self.r1 - self.r0
        b0 = (col0 // self.block) * self.blk
        self.ops.gemm_packed(mloc, col1 - col0, self.k, pa, self.packed_b_full[b0:],
                             C_hi=C_hi[:, col0:col1], C_lo=C_lo[:, col0:col1],
                             flags=None if flags is None else flags[:, col0:col1])
        self.launches += count()

    def __call__(self, A_hi_rows, A_lo_rows, B_hi_slab, B_lo_slab, C_hi=None, C_lo=None,
                 flags=None, events=None):
        """A_*_rows: this rank's rows (r1-r0) x k.  B_*_slab: k x (c1-c0).
        Returns this rank's (C_hi, C_lo, flags) rows.  `events`, if given, is a
        list of 4 CUDA events recorded at the ends of the phases `phase_names`."""
        mloc = self.r1 - self.r0
        count = getattr(self.ops, "launch_count", None) or (lambda: 0)
        self.launches = 0
        if C_hi is None:
            C_hi = torch.empty((mloc, self.n), dtype=torch.float64, device=self.device)
        if C_lo is None:
            C_lo = torch.empty((mloc, self.n), dtype=torch.float64, device=self.device)
        if flags is None:
            flags = torch.empty((mloc, self.n), dtype=torch.uint8, device=self.device)
        self.packed_a = self.ops.pack_a(A_hi_rows, A_lo_rows, packed=self.packed_a)
        self.launches += count()
        rec = (lambda i: events[i].record()) if events else (lambda i: None)
        rec(0)
        w = self.c1 - self.c0
        if self.world == 1:
            self._pack_slab(0, B_hi_slab, B_lo_slab, count)
            rec(1)
            rec(2)
            self._gemm_cols(self.packed_a, 0, self.n, C_hi, C_lo, flags, count)
            rec(3)
            return C_hi, C_lo, flags
        if self.p2p:
            return self._call_p2p(A_hi_rows, A_lo_rows, B_hi_slab, B_lo_slab, C_hi, C_lo, flags,
                                  rec, count)
        if self.raw:
            mine = self.raw_full[self.rank]
            if w > 0:
                mine[0, :, :w].copy_(B_hi_slab)
                mine[1, :, :w].copy_(B_lo_slab)
        if self.overlap:
            # own slab first: packed locally, multiplied while the exchange runs
            self._pack_slab(self.rank, B_hi_slab, B_lo_slab, count)
            rec(1)
            if self.raw:
                work = self._all_gather(self.raw_full.view(-1), self.raw_full[self.rank].view(-1),
                                        async_op=True)
            else:
                work = self._all_gather(self.packed_b_full, self.own, async_op=True)
            self._gemm_cols(self.packed_a, self.c0, self.c1, C_hi, C_lo, flags, count)
            rec(2)
            work.wait()  # the current stream waits for the exchange
            if self.raw:
                for r in range(self.world):
                    a0, a1 = self.slabs[r]
                    if r != self.rank and a1 > a0:
                        self._pack_slab(r, self.raw_full[r, 0, :, :a1 - a0],
                                        self.raw_full[r, 1, :, :a1 - a0], count)
            self._gemm_cols(self.packed_a, self.c1, self.n, C_hi, C_lo, flags, count)
            self._gemm_cols(self.packed_a, 0, self.c0, C_hi, C_lo, flags, count)
            rec(3)
            return C_hi, C_lo, flags
        # serial exchange: all of B gathered first, then one GEMM over all columns
        if self.raw:
            self._all_gather(self.raw_full.view(-1), self.raw_full[self.rank].view(-1))
            rec(1)
            for r in range(self.world):
                a0, a1 = self.slabs[r]
                if a1 > a0:
                    self._pack_slab(r, self.raw_full[r, 0, :, :a1 - a0],
                                    self.raw_full[r, 1, :, :a1 - a0], count)
            rec(2)
        else:
            self._pack_slab(self.rank, B_hi_slab, B_lo_slab, count)
            rec(1)
            self._all_gather(self.packed_b_full, self.own)
            rec(2)
        self._gemm_cols(self.packed_a, 0, self.n, C_hi, C_lo, flags, count)
        rec(3)
        return C_hi, C_lo, flags

    def _call_p2p(self, A_hi_rows, A_lo_rows, B_hi_slab, B_lo_slab, C_hi, C_lo, flags, rec,
                  count):
        """gather = "p2p" (see __init__).  A's pack is already enqueued."""
        cur = torch.cuda.current_stream(self.device)
        # every rank has finished pulling the slabs of the previous call before
        # any rank overwrites its own slab (host waits for its own copy streams)
        if self.copies_pending:
            for ev in self.copy_done:
                ev.synchronize()
        dist.barrier(group=self.cpu_group)
        self._pack_slab(self.rank, B_hi_slab, B_lo_slab, count)
        rec(1)
        packed = torch.cuda.Event()
        packed.record(cur)
        packed.synchronize()  # own slab packed (also: the previous call's GEMMs are done)
        dist.barrier(group=self.cpu_group)  # every rank's own slab is packed
        self._gemm_cols(self.packed_a, self.c0, self.c1, C_hi, C_lo, flags, count)
        rec(2)
        order = [(self.rank + i) % self.world for i in range(1, self.world)]
        for i, q in enumerate(order):  # copy-engine pulls, two streams, neighbours first
            a0, a1 = self.slabs[q]
            if a1 <= a0:
                continue
            cs = self.copy_streams[i % len(self.copy_streams)]
            off = q * self.chunk
            self._casc.casc_copy_async(self._ipc_ptr + off, self.peer_ptrs[q] + off,
                                       self._used(a0, a1), stream=cs)
            self.slab_events[q].record(cs)
        for ev, cs in zip(self.copy_done, self.copy_streams):
            ev.record(cs)
        self.copies_pending = True
        for q in order:  # each slab's columns as soon as that slab has landed
            a0, a1 = self.slabs[q]
            if a1 <= a0:
                continue
            cur.wait_event(self.slab_events[q])
            self._gemm_cols(self.packed_a, a0, a1, C_hi, C_lo, flags, count)
        rec(3)
        return C_hi, C_lo, flags

    def close(self):
        """Release the peer mappings and the exported buffer (p2p; collective)."""
        if not self.p2p or self._ipc_ptr is None:
            return
        torch.cuda.synchronize(self.device)
        if self.copies_pending:
            for ev in self.copy_done:
                ev.synchronize()
        dist.barrier(group=self.cpu_group)  # no rank still copies from a peer
        for ptr in self.peer_ptrs.values():
            self._casc.casc_ipc_close(ptr)
        dist.barrier(group=self.cpu_group)  # every mapping closed before the frees
        self.packed_b_full = None
        self.own = None
        self._casc.casc_ipc_free(self._ipc_ptr)
        self._ipc_ptr = None
