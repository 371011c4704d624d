"""Bucket-range sharding of one logical PIR server over the GPUs of one box
(the paper defers this).

One process per GPU (torchrun). Rank g holds buckets [lo_g, hi_g) (multiples of
8, so every shard reads whole query bytes) and produces a partial answer for
every request; answers are XOR-linear, so the full answer is the XOR of the
partials — the reference's ``pir::reconstruct`` / leader ``contribute``
semantics (pir.cpp:54-73, node.cpp:350-378). NCCL has no XOR reduction, so the
exchange is our own: every rank maps its peers' partial buffers through CUDA IPC
(NVLink / NVSwitch peer loads) and the K4 kernel XOR-reduces the rows it owns
(reduce-scatter: rank g owns requests [g*B/G, (g+1)*B/G)). The mask pad (K3) is
applied exactly once, after the reduce, by the owner.

Fused mode (B >= 2048, the 9-bucket quad-table M4RM kernel 8): the reduce disappears
into the scan. Every owner first initialises its rows (mask pad or zero); then
each rank's scan kernel accumulates the segment partials of every (request
tile, column tile) in a local buffer and the tile's last segment pushes the
finished rows straight into their owners' buffers over NVLink (64-bit
system-scope XOR reductions) while other tiles are still scanning. Per rank and
batch that is B*S bytes, (G-1)/G of them remote — the volume of a
reduce-scatter, overlapped with the scan (``Store.peer_stats`` counts it).

Control plane (handle exchange, barriers) goes through ``torch.distributed``; the
data plane is peer memory only.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous bucket ranges and request-row ownership for G shards."""

    buckets: int
    world: int

    def bucket_range(self, rank: int) -> tuple[int, int]:
        groups = (self.buckets + 7) // 8
        lo = (groups * rank // self.world) * 8
        hi = (groups * (rank + 1) // self.world) * 8
        return lo, min(hi, self.buckets)

    def row_range(self, rank: int, batch: int) -> tuple[int, int]:
        return batch * rank // self.world, batch * (rank + 1) // self.world

    def ranges(self):
        return [self.bucket_range(r) for r in range(self.world)]


def xor_reduce_scatter_reference(partials: list[np.ndarray], plan: ShardPlan, rank: int) -> np.ndarray:
    """Host model of what rank `rank` ends with after the exchange (used by the
    CPU gloo tests to check the plan; never called on the product path)."""
    B = partials[0].shape[0]
    r0, r1 = plan.row_range(rank, B)
    acc = partials[rank][r0:r1].copy()
    for g, p in enumerate(partials):
        if g != rank:
            acc ^= p[r0:r1]
    return acc


class ShardedScan:
    """Per-rank driver: local shard scan + peer XOR reduce-scatter (+ mask)."""

    def __init__(self, xp, torch, dist, N: int, S: int, B: int, device: int, fused: bool | None = None):
        self.xp, self.torch, self.dist = xp, torch, dist
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.plan = ShardPlan(N, self.world)
        self.N, self.S, self.B, self.device = N, S, B, device
        lo, hi = self.plan.bucket_range(self.rank)
        self.store = xp.Store(N, S, lo, hi, device=device)
        # a whole allocation: peers map it through CUDA IPC (handles name allocation bases)
        self._pbuf = xp.DeviceBuffer(B * S, device)
        self.partial = torch.as_tensor(self._pbuf, device=f"cuda:{device}").view(B, S)
        self.r0, self.r1 = self.plan.row_range(self.rank, B)
        self.peers: list[int] = []
        self.src_ptrs = None
        self.fused = (B >= 2048 and S % 32 == 0) if fused is None else bool(fused)
        self._exchange_handles()

    def _exchange_handles(self):
        xp, torch, dist = self.xp, self.torch, self.dist
        h = xp.ipc_handle(self.partial.data_ptr(), self.device)
        handles: list = [None] * self.world
        dist.all_gather_object(handles, h)
        self.peer_base = []
        self.out_ptrs = []  # every rank's answer buffer, rank order (fused mode)
        for g, hg in enumerate(handles):
            if g == self.rank:
                self.out_ptrs.append(self.partial.data_ptr())
                continue
            self.peer_base.append(xp.ipc_open(hg, self.device))
            self.out_ptrs.append(self.peer_base[-1])
        self.row_bounds = [self.plan.row_range(g, self.B)[0] for g in range(self.world)] + [self.B]
        row = self.r0 * self.S
        ptrs = [p + row for p in self.peer_base]
        self.src_ptrs = torch.tensor(ptrs if ptrs else [0], dtype=torch.int64, device=f"cuda:{self.device}")
        self.nsrc = len(ptrs)

    def close(self):
        for p in self.peer_base:
            self.xp.ipc_close(p, self.device)
        self.peer_base = []
        self.store.close()
        self.partial = None
        self._pbuf.close()

    def step(self, d_seeds, stream=None, d_mask=None):
        """One batch: partial scan of this shard, barrier, reduce own rows from
        peers, barrier. Returns the view of this rank's final rows."""
        xp, torch, dist = self.xp, self.torch, self.dist
        if self.fused:
            return self._step_fused(d_seeds, stream, d_mask)
        self.store.answer_batch_seeded_dev(d_seeds, self.B, self.partial, stream=stream)
        own = self.partial[self.r0:self.r1]
        if self.world > 1:
            torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()
            dist.barrier()
            xp.xor_reduce_dev(own, [0] * self.nsrc, (self.r1 - self.r0) * self.S, device=self.device,
                              stream=stream, d_ptr_array=self.src_ptrs)
        if d_mask is not None:
            xp.mask_dev(own, d_mask[self.r0:self.r1], self.r1 - self.r0, self.S, device=self.device,
                        stream=stream)
        if self.world > 1:
            torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()
            dist.barrier()  # peers finished reading our partial before it is overwritten
        return own

    def _sync_barrier(self, stream):
        torch = self.torch
        torch.cuda.current_stream(self.device).synchronize() if stream is None else stream.synchronize()
        if self.world > 1:
            self.dist.barrier()

    def _step_fused(self, d_seeds, stream, d_mask):
        """Owner init -> barrier -> scan whose epilogue XORs into the owners'
        buffers -> barrier. The second barrier also guarantees no peer still
        writes our rows when the next step re-initialises them."""
        xp = self.xp
        xp.init_rows_dev(self.partial, self.r0, self.r1, self.S, d_mask, device=self.device, stream=stream)
        self._sync_barrier(stream)
        self.store.answer_batch_seeded_peer_dev(d_seeds, self.B, self.out_ptrs, self.row_bounds, self.rank,
                                                stream=stream)
        self._sync_barrier(stream)
        return self.partial[self.r0:self.r1]
