"""Multi-GPU domain decomposition of the block rows.

One process per GPU.  Block rows are split into contiguous ranges (z-slabs of
cells for the Cartesian configs); a rank's local operator keeps its own rows
with columns renumbered [owned blocks | ghost blocks], ghosts sorted by
global block id (so each owner's ghosts are one contiguous range).

`HaloPlan` is built once from the local column pattern: ranks exchange the
ghost lists they need (setup, all_gather_object), then every `exchange`
posts grouped P2P sends of packed owned blocks (xdg_gather_blocks) and
receives straight into the ghost tail of the extended vector
(torch.distributed over NCCL on NVLink; gloo on CPU for the tests).  The SpMV
overlaps the transfer: interior rows (no ghost columns) run while the halo
is in flight, boundary rows after the wait.

Reductions (dots/norms of the Krylov/RM loops) are rank-local partial sums
reduced with one all_reduce per scalar batch (`allreduce_sum`).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def owners_of(row_starts: np.ndarray, ids: np.ndarray) -> np.ndarray:
    return np.searchsorted(row_starts, ids, side="right") - 1


class HaloPlan:
    def __init__(self, row_starts, ghost_ids, rank: int, world: int, N: int,
                 device, group=None):
        self.rank, self.world, self.N = rank, world, N
        self.device = device
        self.group = group
        rs = np.asarray(row_starts, np.int64)
        self.row0, self.row1 = int(rs[rank]), int(rs[rank + 1])
        self.nloc = self.row1 - self.row0
        g = np.asarray(ghost_ids, np.int64)
        if len(g) and (np.any(np.diff(g) <= 0)):
            raise ValueError("ghost ids must be sorted and unique")
        own = owners_of(rs, g)
        if np.any(own == rank):
            raise ValueError("a ghost block is owned by this rank")
        self.nghost = len(g)
        # receive ranges inside the ghost tail, per owner
        self.recvs = {}
        for q in np.unique(own):
            pos = np.flatnonzero(own == q)
            self.recvs[int(q)] = (int(pos[0]), int(pos[-1]) + 1)
        requests = {int(q): g[own == q] for q in np.unique(own)}
        gathered = [None] * world
        if world > 1:
            dist.all_gather_object(gathered, requests, group=group)
        else:
            gathered = [requests]
        self.sends = {}
        for p in range(world):
            want = gathered[p].get(rank) if gathered[p] else None
            if p != rank and want is not None and len(want):
                local = np.asarray(want, np.int64) - self.row0
                if np.any(local < 0) or np.any(local >= self.nloc):
                    raise ValueError("peer requested a block this rank does not own")
                self.sends[p] = torch.from_numpy(local.astype(np.int32)).to(device)
        self.sendbufs = {p: torch.empty(len(i) * N, dtype=torch.float64, device=device)
                         for p, i in self.sends.items()}

    @property
    def halo_bytes(self) -> int:
        return 8 * self.N * (self.nghost + sum(len(i) for i in self.sends.values()))

    def _pack(self, x_ext: torch.Tensor):
        if x_ext.is_cuda:
            from .device import Context
            from . import _native as nat

            ctx = Context.get(x_ext.device)
            for p, idx in self.sends.items():
                nat.check(ctx.lib.xdg_gather_blocks(
                    idx.numel(), self.N, idx.data_ptr(), x_ext.data_ptr(),
                    self.sendbufs[p].data_ptr(), ctx.stream), "gather_blocks")
        else:  # CPU (gloo) path of the tests: host-side packing
            xv = x_ext[: self.nloc * self.N].view(-1, self.N)
            for p, idx in self.sends.items():
                self.sendbufs[p].copy_(xv[idx.long()].reshape(-1))

    def _host_staged(self, x_ext) -> bool:
        """gloo cannot move CUDA tensors point to point: stage through host
        memory (the tests run several gloo ranks on one GPU)."""
        return x_ext.is_cuda and dist.get_backend(self.group) == "gloo"

    def start(self, x_ext: torch.Tensor):
        """Post the exchange; returns a pending handle (wait with `finish`)."""
        if self.world == 1 or (not self.sends and not self.recvs):
            return []
        self._pack(x_ext)
        ops, post = [], []
        base = self.nloc * self.N
        staged = self._host_staged(x_ext)
        for q, (lo, hi) in sorted(self.recvs.items()):
            dst = x_ext[base + lo * self.N: base + hi * self.N]
            if staged:
                buf = torch.empty(dst.numel(), dtype=dst.dtype)
                post.append((dst, buf))
                dst = buf
            ops.append(dist.P2POp(dist.irecv, dst, q, group=self.group))
        for p, _ in sorted(self.sends.items()):
            src = self.sendbufs[p].cpu() if staged else self.sendbufs[p]
            ops.append(dist.P2POp(dist.isend, src, p, group=self.group))
        return (dist.batch_isend_irecv(ops), post)

    @staticmethod
    def finish(pending):
        if not pending:
            return
        reqs, post = pending
        for r in reqs:
            r.wait()
        for dst, buf in post:
            dst.copy_(buf)

    def exchange(self, x_ext: torch.Tensor):
        self.finish(self.start(x_ext))

    def reverse(self, ghost_vals: torch.Tensor) -> dict:
        """Transpose of `exchange`: send the values this rank holds for its
        ghost blocks (ghost_vals, (nghost * N,)) back to their owners;
        returns {source rank: received values for self.sends[source]}."""
        if self.world == 1:
            return {}
        staged = ghost_vals.is_cuda and dist.get_backend(self.group) == "gloo"
        ops, bufs = [], {}
        for p, idx in sorted(self.sends.items()):
            buf = torch.empty(idx.numel() * self.N, dtype=ghost_vals.dtype,
                              device="cpu" if staged else ghost_vals.device)
            bufs[p] = buf
            ops.append(dist.P2POp(dist.irecv, buf, p, group=self.group))
        for q, (lo, hi) in sorted(self.recvs.items()):
            src = ghost_vals[lo * self.N: hi * self.N]
            ops.append(dist.P2POp(dist.isend, src.cpu() if staged else src, q,
                                  group=self.group))
        for r in dist.batch_isend_irecv(ops) if ops else []:
            r.wait()
        if staged:
            bufs = {p: b.to(ghost_vals.device) for p, b in bufs.items()}
        return bufs


def split_interior(row_ptr: np.ndarray, col: np.ndarray, nloc: int):
    """(a, b): rows [a, b) reference no ghost column; rows outside are the
    boundary.  Falls back to (0, 0) if the interior is not contiguous."""
    nrows = len(row_ptr) - 1
    rows_of = np.repeat(np.arange(nrows), np.diff(row_ptr))
    bnd = np.zeros(nrows, bool)
    bnd[rows_of[col >= nloc]] = True
    if not bnd.any():
        return 0, nrows
    idx = np.flatnonzero(bnd)
    mid = nrows // 2
    lo = idx[idx < mid]
    hi = idx[idx >= mid]
    a = int(lo[-1]) + 1 if len(lo) else 0
    b = int(hi[0]) if len(hi) else nrows
    if a >= b or bnd[a:b].any():
        return 0, 0
    return a, b


class DistributedSpMV:
    """y_local = (M x)[owned rows] for a slab-partitioned operator: halo
    exchange overlapped with the interior rows."""

    def __init__(self, D, halo: HaloPlan, row_ptr_host=None, col_host=None):
        self.D, self.halo = D, halo
        rp = D.row_ptr.cpu().numpy() if row_ptr_host is None else row_ptr_host
        cl = D.col.cpu().numpy() if col_host is None else col_host
        self.a, self.b = split_interior(np.asarray(rp, np.int64), np.asarray(cl, np.int64),
                                        halo.nloc)

    def __call__(self, x_ext: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        reqs = self.halo.start(x_ext)
        nbr = self.D.nbr
        if self.b > self.a:
            self.D.spmv(x_ext, y, rows=(self.a, self.b))
            HaloPlan.finish(reqs)
            if self.a > 0:
                self.D.spmv(x_ext, y, rows=(0, self.a))
            if self.b < nbr:
                self.D.spmv(x_ext, y, rows=(self.b, nbr))
        else:
            HaloPlan.finish(reqs)
            self.D.spmv(x_ext, y)
        return y


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t
