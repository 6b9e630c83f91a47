"""Multi-GPU GMRES-PMG: one process per GPU, block rows
partitioned in contiguous ranges.

Per rank:
  * the local operator (owned rows, columns [owned | ghosts]) and a HaloPlan;
    every M x is a DistributedSpMV (halo exchange overlapped with the
    interior rows);
  * the degree-separated preconditioner (solvers.py:183-305) split the way
    the method allows: the global low-order system does NOT shard (it couples
    every cell), so its right-hand side is all-gathered and the dense
    factor is applied redundantly on every rank ("replicas only" for that
    stage); the high-order stage is rank-local (fused residual
    + per-cell LU, reading the replicated low-order solution by global cell
    id);
  * Krylov inner products are rank-local partial dots + one all-reduce each
    (MGS keeps the reference's j+1 sequential reductions), so every rank
    holds the same Hessenberg column and takes the same scalar decisions.

Collectives go through torch.distributed: NCCL on device tensors, or gloo
staged through host memory (tests run several gloo ranks on one GPU; no
kernel ever waits on another rank).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from time import perf_counter

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .device import Context, DeviceBSR
from .direct import (
    SPARSE_DIRECT_MIN,
    DeviceDirect,
    SparseDirect,
    dense_from_device_bsr,
)
from .distributed import DistributedSpMV, HaloPlan
from .errors import SingularSystemError
from .factor import batched_factor
from .solvers import SolverConfig, SolverReport, space_dimension

F64 = torch.float64
I32 = torch.int32


class Comm:
    """Sum all-reduce / all-gather over a process group (NCCL direct, gloo
    host-staged)."""

    def __init__(self, group=None):
        self.group = group
        self.on = dist.is_available() and dist.is_initialized()
        self.world = dist.get_world_size(group) if self.on else 1
        self.rank = dist.get_rank(group) if self.on else 0
        self.host = self.on and dist.get_backend(group) == "gloo"

    def allreduce_(self, t: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            return t
        if self.host:
            h = t.cpu()
            dist.all_reduce(h, group=self.group)
            t.copy_(h)
        else:
            dist.all_reduce(t, group=self.group)
        return t

    def allgather_cat(self, local: torch.Tensor, counts) -> torch.Tensor:
        """Concatenation over ranks of variable-length 1-D tensors."""
        if self.world == 1:
            return local
        mx = int(max(counts))
        pad = torch.zeros(mx, dtype=local.dtype, device=local.device)
        pad[: local.numel()] = local
        if self.host:
            pad = pad.cpu()
        parts = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(parts, pad, group=self.group)
        out = torch.cat([p[:c] for p, c in zip(parts, counts)])
        return out.to(local.device)


def balanced_row_starts(nbr: int, world: int) -> np.ndarray:
    return np.array([(nbr * r) // world for r in range(world + 1)], np.int64)


@dataclass
class LocalOperator:
    D: DeviceBSR          # local rows, columns [owned | ghosts]
    gcol: np.ndarray      # global block column of every local block
    ghosts: np.ndarray    # global ids of the ghost blocks (sorted)
    r0: int
    r1: int


def local_operator(rp, col, val, N, row_starts, rank, ctx) -> LocalOperator:
    r0, r1 = int(row_starts[rank]), int(row_starts[rank + 1])
    k0, k1 = int(rp[r0]), int(rp[r1])
    nloc = r1 - r0
    gcol = np.asarray(col[k0:k1], np.int64)
    owned = (gcol >= r0) & (gcol < r1)
    ghosts = np.unique(gcol[~owned])
    lcol = np.where(owned, gcol - r0, 0)
    lcol[~owned] = nloc + np.searchsorted(ghosts, gcol[~owned])
    D = DeviceBSR.from_arrays(np.asarray(rp[r0:r1 + 1]) - k0, lcol, val[k0:k1], N,
                              nloc + len(ghosts), ctx)
    return LocalOperator(D, gcol, ghosts, r0, r1)


class DistPmg:
    """Degree-separated preconditioner over ALL cells (the GMRES-PMG cell
    set, solvers.py:800), distributed: the global low-order solve through
    the multifrontal factor whose elimination subtrees are mapped to the
    ranks (each rank factors and stores only its subtrees plus the shared
    top fronts: multifrontal.proportional_map), or a replicated dense factor
    for small systems; the high-order stage is rank-local."""

    def __init__(self, rp, col, val, N, m, op: LocalOperator, row_starts, comm: Comm, ctx):
        self.ctx, self.comm, self.op = ctx, comm, op
        self.N, self.m = N, m
        dev = ctx.device
        nbr = len(rp) - 1
        nloc = op.r1 - op.r0
        self.nloc = nloc
        self.counts = [int(row_starts[q + 1] - row_starts[q]) * m for q in range(comm.world)]
        # low-order factor from the global blocks' (:m, :m) parts
        lo_val = np.ascontiguousarray(np.asarray(val)[:, :m, :m])
        Dlo = DeviceBSR.from_arrays(rp, col, lo_val, m, nbr, ctx)
        mode = os.environ.get("XDG_LOW_ORDER", "auto")
        sparse = mode == "sparse" or (mode != "dense" and nbr * m > SPARSE_DIRECT_MIN)
        try:
            if sparse:  # multifrontal (cfg2: 336,610 unknowns), subtrees over the ranks
                self.low = SparseDirect(Dlo, ctx, "low-order system", comm=comm)
            else:
                A = dense_from_device_bsr(Dlo)
                self.low = DeviceDirect(A, ctx, "low-order system")
                del A
        except SingularSystemError as exc:
            raise SingularSystemError("low-order system is singular") from exc
        del Dlo
        self.blo_own = torch.empty(nloc * m, dtype=F64, device=dev)
        self.xlo = torch.empty(nbr * m, dtype=F64, device=dev)
        self.rows_global = torch.arange(op.r0, op.r1, dtype=I32, device=dev)
        self.has_high = m < N
        if self.has_high:
            nh = N - m
            lrp = np.asarray(rp[op.r0:op.r1 + 1]) - int(rp[op.r0])
            rows_of = np.repeat(np.arange(nloc), np.diff(lrp))
            isdiag = op.gcol == rows_of + op.r0
            diag_k = np.full(nloc, -1, np.int64)
            diag_k[rows_of[isdiag]] = np.flatnonzero(isdiag)
            if np.any(diag_k < 0):
                raise SingularSystemError(
                    f"cell {int(op.r0 + np.flatnonzero(diag_k < 0)[0])} has no diagonal block")
            H = torch.empty(nloc * nh * nh, dtype=F64, device=dev)
            up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)  # noqa: E731
            nat.check(ctx.lib.xdg_pmg_gather_high(
                nloc, N, m, up(np.arange(nloc), I32).data_ptr(), up(diag_k, I32).data_ptr(),
                op.D.val_t.data_ptr(), H.data_ptr(), ctx.stream), "pmg_gather_high")
            hoff = np.arange(nloc, dtype=np.int64) * nh
            hperm, _, info = batched_factor(ctx, H, hoff * nh, np.full(nloc, nh, np.int32),
                                            invert=False, perm_off=hoff)
            bad = torch.nonzero(info[:nloc])
            if bad.numel():
                c = op.r0 + int(bad[0])
                raise SingularSystemError(f"high-order block of cell {c} is singular")
            self.HLU = torch.empty_like(H)
            nat.check(ctx.lib.xdg_blocks_transpose(nloc, nh, H.data_ptr(),
                                                   self.HLU.data_ptr(), ctx.stream), "transpose")
            self.hperm = hperm
            self.wi_ptr = op.D.row_ptr
            self.wi_blk = torch.arange(op.D.nnzb, dtype=I32, device=dev)
            self.wi_lcol = up(op.gcol, I32)                  # global cell -> xlo
            self.wi_cell = torch.arange(nloc, dtype=I32, device=dev)   # local b / out
            self.wi_lrow = self.rows_global                   # own x_lo, global id
            self.wi_xlo = torch.zeros(nloc, dtype=torch.int64, device=dev)
            self.wi_hidx = self.wi_cell
            self.wi_out = torch.arange(nloc, dtype=torch.int64, device=dev) * N

    def apply(self, b_loc: torch.Tensor, z_loc: torch.Tensor) -> torch.Tensor:
        ctx, N, m = self.ctx, self.N, self.m
        nat.check(ctx.lib.xdg_gather_modes(self.nloc, N, m, b_loc.data_ptr(),
                                           self.blo_own.data_ptr(), ctx.stream), "gather_modes")
        blo = self.comm.allgather_cat(self.blo_own, self.counts)
        self.low.apply(blo, self.xlo)
        if self.has_high:
            nat.check(ctx.lib.xdg_pmg_high(
                self.nloc, N, m, self.wi_ptr.data_ptr(), self.wi_blk.data_ptr(),
                self.wi_lcol.data_ptr(), self.wi_cell.data_ptr(), self.wi_lrow.data_ptr(),
                self.wi_xlo.data_ptr(), self.wi_hidx.data_ptr(), self.wi_out.data_ptr(),
                self.op.D.val_t.data_ptr(), self.HLU.data_ptr(), self.hperm.data_ptr(),
                b_loc.data_ptr(), self.xlo.data_ptr(), z_loc.data_ptr(), ctx.stream),
                "pmg_high")
        else:
            nat.check(ctx.lib.xdg_gather_blocks(self.nloc, N, self.rows_global.data_ptr(),
                                                self.xlo.data_ptr(), z_loc.data_ptr(),
                                                ctx.stream), "gather_blocks")
        return z_loc


def dist_gmres_pmg_solve(rp, col, val, b, config: SolverConfig, *, dim: int,
                         group=None, row_starts=None):
    """Restarted right-preconditioned GMRES (solvers.py:756-846) over the
    ranks of `group`.  rp/col/val: the GLOBAL level matrix (row-major blocks;
    every rank passes the same arrays, each uploads only its rows); b: the
    global right-hand side (numpy).  Returns (x_local numpy, (r0, r1) block
    rows, SolverReport) -- the report is identical on every rank."""
    ctx = Context.get()
    comm = Comm(group)
    val = np.asarray(val)
    N = val.shape[1]
    nbr = len(rp) - 1
    if row_starts is None:
        row_starts = balanced_row_starts(nbr, comm.world)
    t_start = perf_counter()
    op = local_operator(rp, col, val, N, row_starts, comm.rank, ctx)
    halo = HaloPlan(row_starts, op.ghosts, comm.rank, comm.world, N, ctx.device, group)
    spmv = DistributedSpMV(op.D, halo)
    m_lo = min(space_dimension(config.k_lo_scalar, dim), N)
    pmg = DistPmg(rp, col, val, N, m_lo, op, row_starts, comm, ctx)
    dev = ctx.device
    nloc, ng = op.r1 - op.r0, len(op.ghosts)
    L, Le = nloc * N, (nloc + ng) * N
    m = config.gmres_restart
    bl = torch.from_numpy(np.ascontiguousarray(b[op.r0 * N: op.r1 * N], float)).to(dev)
    x = torch.zeros(Le, dtype=F64, device=dev)           # extended (ghosts for M x)
    V = torch.empty(m + 1, L, dtype=F64, device=dev)
    Z = torch.zeros(m, Le, dtype=F64, device=dev)         # SpMV inputs: extended
    w = torch.empty(L, dtype=F64, device=dev)
    r = torch.empty(L, dtype=F64, device=dev)
    sc = torch.zeros(m + 2, dtype=F64, device=dev)
    ycoef = torch.zeros(m, dtype=F64, device=dev)

    def gdot(u, v, out):
        ctx.dot(u, v, out)
        return comm.allreduce_(out)

    def residual():
        spmv(x, w)
        ctx.sub(bl, w, r)
        gdot(r, r, sc[0:1])
        return math.sqrt(float(sc[0].item()))

    beta = residual()
    history, total = [beta], 0
    while beta > config.tolerance and total < config.max_iterations:
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        ctx.scale(beta, r, V[0], invert=True)
        j = 0
        while j < m and total < config.max_iterations:
            total += 1
            pmg.apply(V[j], Z[j, :L])
            spmv(Z[j], w)
            # modified Gram-Schmidt (solvers.py:802-805): step i's axpy fused
            # with step i+1's dot (xdg_axpy_dot), one all-reduce per step
            gdot(V[0], w, sc[0:1])
            for i in range(j + 1):
                nat.check(ctx.lib.xdg_axpy_dot(
                    L, -1.0, sc[i:i + 1].data_ptr(), V[i].data_ptr(), w.data_ptr(),
                    V[i + 1].data_ptr() if i < j else None, sc[i + 1:i + 2].data_ptr(),
                    ctx.ws, ctx.stream), "axpy_dot")
                comm.allreduce_(sc[i + 1:i + 2])
            col_h = sc[: j + 2].cpu().numpy()
            H[: j + 1, j] = col_h[: j + 1]
            H[j + 1, j] = math.sqrt(col_h[j + 1])
            if H[j + 1, j] > 0.0:
                ctx.scale(H[j + 1, j], w, V[j + 1], invert=True)
            else:
                V[j + 1].zero_()
            for i in range(j):
                h_i = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = h_i
            denom = float(np.hypot(H[j, j], H[j + 1, j]))
            if denom == 0.0:
                raise SingularSystemError("preconditioned operator produced a zero column")
            cs[j], sn[j] = H[j, j] / denom, H[j + 1, j] / denom
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[j + 1, j] = 0.0
            est = abs(float(g[j + 1]))
            history.append(est)
            j += 1
            if est <= config.tolerance:
                break
        yv = np.zeros(j)
        for i in range(j - 1, -1, -1):                   # back substitution
            yv[i] = (g[i] - H[i, i + 1:j] @ yv[i + 1:]) / H[i, i]
        ycoef[:j].copy_(torch.from_numpy(-yv))
        nat.check(ctx.lib.xdg_gemv_update2(L, j, Z.data_ptr(), None, Le, ycoef.data_ptr(),
                                           None, x.data_ptr(), None, ctx.stream), "x += Z y")
        beta = residual()
        history[-1] = beta
    torch.cuda.synchronize(dev)
    rep = SolverReport(solver="gmres-pmg", iterations=total,
                       converged=beta <= config.tolerance, final_residual=beta,
                       residual_history=history, time_iterations=perf_counter() - t_start,
                       dofs=nbr * N)
    return x[:L].cpu().numpy(), (op.r0, op.r1), rep


# ===========================================================================
# Multi-GPU orthonormalization multigrid (solvers.py:669-749)
#
# Per level: contiguous block-row partition; M, R (fine rows x coarse cols)
# and R^T (coarse rows x fine cols) as local operators with halos on their
# column spaces.  Schwarz smoother (solvers.py:460-478), owner-computes: the
# global BFS partition is built identically on every rank, each extended
# block is owned by the rank owning its first core cell, a rank smooths its
# blocks on the union U of their cells (residual gathered for foreign cells,
# one batched PmgPlan), and the undamped partial sums for foreign cells go
# back to their owners, which add all ranks' partials in rank order (= block
# order; a roundoff-level reassociation of the reference's sum) and divide by
# the damping.  RM reductions are all-reduced (5 per rm_step); the coarsest
# level is solved redundantly after an all-gather of its right-hand side.

def _transpose_bsr(rp, col, val, ncols):
    """BSR arrays of the block transpose (rows sorted, blocks transposed)."""
    nbr = len(rp) - 1
    rows = np.repeat(np.arange(nbr), np.diff(rp))
    order = np.lexsort((rows, col))
    trp = np.zeros(ncols + 1, np.int64)
    np.cumsum(np.bincount(col, minlength=ncols), out=trp[1:])
    return trp, rows[order], np.ascontiguousarray(np.transpose(val[order], (0, 2, 1)))


def local_rect_operator(rp, col, val, N, row_starts, col_starts, rank, ctx) -> LocalOperator:
    """Rows of this rank (row partition) with columns renumbered [owned in
    the column partition | ghosts]."""
    r0, r1 = int(row_starts[rank]), int(row_starts[rank + 1])
    c0, c1 = int(col_starts[rank]), int(col_starts[rank + 1])
    k0, k1 = int(rp[r0]), int(rp[r1])
    ncl = c1 - c0
    gcol = np.asarray(col[k0:k1], np.int64)
    owned = (gcol >= c0) & (gcol < c1)
    ghosts = np.unique(gcol[~owned])
    lcol = np.where(owned, gcol - c0, 0)
    lcol[~owned] = ncl + np.searchsorted(ghosts, gcol[~owned])
    D = DeviceBSR.from_arrays(np.asarray(rp[r0:r1 + 1]) - k0, lcol, val[k0:k1], N,
                              ncl + len(ghosts), ctx)
    return LocalOperator(D, gcol, ghosts, r0, r1)


class _DistOp:
    """y_local = A x for a row-partitioned operator with a halo on x."""

    def __init__(self, op: LocalOperator, col_starts, comm, ctx, group):
        self.op, self.ctx = op, ctx
        self.N = op.D.N
        self.halo = HaloPlan(col_starts, op.ghosts, comm.rank, comm.world, self.N,
                             ctx.device, group)
        self.spmv = DistributedSpMV(op.D, self.halo)
        self.ext = torch.zeros(op.D.nbc * self.N, dtype=F64, device=ctx.device)
        self.ncol_own = self.halo.nloc

    def __call__(self, x_own: torch.Tensor, y: torch.Tensor) -> torch.Tensor:
        self.ext[: self.ncol_own * self.N].copy_(x_own)
        return self.spmv(self.ext, y)


class _DistSchwarz:
    def __init__(self, rp, col, val, N, part, m, row_starts, comm, ctx, group):
        from .pmg import PmgPlan

        self.ctx, self.comm, self.N = ctx, comm, N
        dev = ctx.device
        r0, r1 = int(row_starts[comm.rank]), int(row_starts[comm.rank + 1])
        self.nloc = r1 - r0
        owner = np.searchsorted(row_starts, [c[0] for c in part.cores], side="right") - 1
        mine = [i for i in range(len(part.block_rows)) if owner[i] == comm.rank]
        U = np.unique(np.concatenate([np.asarray(part.block_rows[i]) for i in mine])) \
            if mine else np.zeros(0, np.int64)
        self.U = U
        own = (U >= r0) & (U < r1)
        foreign = U[~own]
        # residual gather: [owned cells | foreign cells of U] then U order
        self.halo = HaloPlan(row_starts, foreign, comm.rank, comm.world, N, dev, group)
        self.r_ext = torch.zeros((self.nloc + len(foreign)) * N, dtype=F64, device=dev)
        pos = np.where(own, U - r0, self.nloc + np.searchsorted(foreign, U))
        self.u_from_ext = torch.from_numpy(pos.astype(np.int32)).to(dev)
        self.rU = torch.zeros(max(len(U), 1) * N, dtype=F64, device=dev)
        self.zU = torch.zeros(max(len(U), 1) * N, dtype=F64, device=dev)
        self.own_u = torch.from_numpy(np.flatnonzero(own).astype(np.int32)).to(dev)
        self.own_dst = torch.from_numpy((U[own] - r0).astype(np.int32)).to(dev)
        self.foreign_u = torch.from_numpy(np.flatnonzero(~own).astype(np.int32)).to(dev)
        self.foreign_vals = torch.zeros(max(len(foreign), 1) * N, dtype=F64, device=dev)
        self.damp = torch.from_numpy(np.ascontiguousarray(
            part.damping[r0 * N: r1 * N], float)).to(dev)
        self.tmp = torch.zeros(self.nloc * N, dtype=F64, device=dev)
        self.plan = None
        if mine:
            # operator restricted to U x U (renumbered), the blocks' local cells
            loc = np.full(len(rp) - 1, -1, np.int64)
            loc[U] = np.arange(len(U))
            rows, cols, ks = [], [], []
            for u, c in enumerate(U):
                kk = np.arange(rp[c], rp[c + 1])
                lc = loc[col[kk]]
                keep = lc >= 0
                rows.append(np.full(keep.sum(), u))
                cols.append(lc[keep])
                ks.append(kk[keep])
            rows, cols, ks = np.concatenate(rows), np.concatenate(cols), np.concatenate(ks)
            urp = np.zeros(len(U) + 1, np.int64)
            np.cumsum(np.bincount(rows, minlength=len(U)), out=urp[1:])
            DU = DeviceBSR.from_arrays(urp, cols, val[ks], N, len(U), ctx)
            sets = [loc[np.asarray(part.block_rows[i])] for i in mine]
            self.plan = PmgPlan(DU, sets, m, damping=None, combine=True)

    def __call__(self, r_own: torch.Tensor, z_own: torch.Tensor) -> torch.Tensor:
        ctx, N = self.ctx, self.N
        lib, st = ctx.lib, ctx.stream
        self.r_ext[: self.nloc * N].copy_(r_own)
        self.halo.exchange(self.r_ext)
        nU = len(self.U)
        if self.plan is not None:
            nat.check(lib.xdg_gather_blocks(nU, N, self.u_from_ext.data_ptr(),
                                            self.r_ext.data_ptr(), self.rU.data_ptr(), st),
                      "gather r_U")
            self.plan.apply(self.rU, self.zU)      # undamped partial sums on U
            nat.check(lib.xdg_gather_blocks(self.foreign_u.numel(), N,
                                            self.foreign_u.data_ptr(), self.zU.data_ptr(),
                                            self.foreign_vals.data_ptr(), st), "pack")
        recv = self.halo.reverse(self.foreign_vals)
        z_own.zero_()
        for q in range(self.comm.world):       # rank order == block order
            if q == self.comm.rank:
                if self.plan is not None and self.own_u.numel():
                    nat.check(lib.xdg_gather_blocks(self.own_u.numel(), N,
                                                    self.own_u.data_ptr(),
                                                    self.zU.data_ptr(), self.tmp.data_ptr(),
                                                    st), "own partial")
                    nat.check(lib.xdg_scatter_add_blocks(self.own_dst.numel(), N,
                                                         self.own_dst.data_ptr(),
                                                         self.tmp.data_ptr(),
                                                         z_own.data_ptr(), st), "add own")
            elif q in recv:
                idx = self.halo.sends[q]
                nat.check(lib.xdg_scatter_add_blocks(idx.numel(), N, idx.data_ptr(),
                                                     recv[q].data_ptr(), z_own.data_ptr(),
                                                     st), "add peer partials")
        ctx.div(z_own, self.damp, z_own)
        return z_own


class _DistRm:
    """RmState + rm_step (solvers.py:485-625) over row-distributed vectors."""

    def __init__(self, n, max_columns, M: _DistOp, comm, ctx):
        self.n, self.cap, self.M, self.comm, self.ctx = n, max_columns, M, comm, ctx
        dev = ctx.device
        self.W = torch.empty(max_columns, n, dtype=F64, device=dev)
        self.Z = torch.empty(max_columns, n, dtype=F64, device=dev)
        v = torch.zeros(8, n, dtype=F64, device=dev)
        self.vec = v
        self.x0, self.r0, self.y, self.My, self.My_new, self.Mz, self.x, self.r = v
        self.coeff = torch.zeros(3, max(max_columns, 1), dtype=F64, device=dev)
        self.sc = torch.zeros(8, dtype=F64, device=dev)
        self.gws = torch.zeros((int(ctx.lib.xdg_gemv_t_workspace_bytes(max(max_columns, 1)))
                                + 7) // 8, dtype=F64, device=dev)

    def init(self, x, r):
        self.x0.copy_(x)
        self.r0.copy_(r)
        self.x.copy_(x)      # current point / true residual (RmState.current())
        self.r.copy_(r)
        self.y.zero_()
        self.My.zero_()
        self.ctx.dot(self.r0, self.r0, self.sc[7:8])
        self.comm.allreduce_(self.sc[7:8])
        self.best = math.sqrt(float(self.sc[7].item()))
        self.ncols = 0

    def _restart(self):
        nat.check(self.ctx.lib.xdg_rm_restart_vec(
            self.n, self.x0.data_ptr(), self.r0.data_ptr(), self.y.data_ptr(),
            self.My.data_ptr(), self.x.data_ptr(), self.r.data_ptr(), self.ctx.stream),
            "rm_restart")
        self.ncols = 0   # best unchanged: it is ||r0 - My|| of the new r0

    def step(self, zc):
        ctx, lib, st, n, sc = self.ctx, self.ctx.lib, self.ctx.stream, self.n, self.sc
        if self.ncols >= self.cap:
            self._restart()
        col = self.ncols
        z, w = self.Z[col], self.W[col]
        z.copy_(zc)
        self.M(z, w)
        ctx.dot(w, w, sc[0:1])
        if col > 0:
            c1, c2, cs = self.coeff[0], self.coeff[1], self.coeff[2]
            nat.check(lib.xdg_gemv_t(n, col, self.W.data_ptr(), n, w.data_ptr(),
                                     c1.data_ptr(), self.gws.data_ptr(), st), "gemv_t")
            self.comm.allreduce_(c1[:col])
            nat.check(lib.xdg_gemv_update2(n, col, self.W.data_ptr(), None, n, c1.data_ptr(),
                                           None, w.data_ptr(), None, st), "update")
            nat.check(lib.xdg_gemv_t(n, col, self.W.data_ptr(), n, w.data_ptr(),
                                     c2.data_ptr(), self.gws.data_ptr(), st), "gemv_t")
            self.comm.allreduce_(c2[:col])
            nat.check(lib.xdg_add_small(col, c1.data_ptr(), c2.data_ptr(), cs.data_ptr(), st),
                      "c1+c2")
            nat.check(lib.xdg_gemv_update2(n, col, self.W.data_ptr(), self.Z.data_ptr(), n,
                                           c2.data_ptr(), cs.data_ptr(), w.data_ptr(),
                                           z.data_ptr(), st), "update2")
        ctx.dot(w, w, sc[1:2])
        self.comm.allreduce_(sc[0:2])
        nat.check(lib.xdg_rm_normalize(n, sc[1:2].data_ptr(), w.data_ptr(), z.data_ptr(), st),
                  "rm_normalize")
        ctx.dot(w, self.r0, sc[2:3])
        self.comm.allreduce_(sc[2:3])
        self.M(z, self.Mz)
        nat.check(lib.xdg_rm_update(n, self.r0.data_ptr(), self.My.data_ptr(),
                                    self.Mz.data_ptr(), sc[2:3].data_ptr(),
                                    self.My_new.data_ptr(), sc[3:4].data_ptr(), ctx.ws, st),
                  "rm_update")
        self.comm.allreduce_(sc[3:4])
        h = sc[0:4].cpu().numpy()
        scale, nw = math.sqrt(h[0]), math.sqrt(h[1])
        if scale == 0.0 or nw <= 1e-13 * scale:
            ctx.lib.xdg_add(n, self.x0.data_ptr(), self.y.data_ptr(), self.x.data_ptr(), st)
            ctx.sub(self.r0, self.My, self.r)
            return
        rho = math.sqrt(h[3])
        if rho > self.best:
            self._restart()
            return
        nat.check(lib.xdg_rm_commit(n, sc[2:3].data_ptr(), z.data_ptr(), self.y.data_ptr(),
                                    self.x0.data_ptr(), self.r0.data_ptr(),
                                    self.My_new.data_ptr(), self.x.data_ptr(),
                                    self.r.data_ptr(), st), "rm_commit")
        self.My, self.My_new = self.My_new, self.My
        self.best = rho
        self.ncols = col + 1


def dist_ortho_mg_solve(hierarchy, b, config: SolverConfig, *, group=None):
    """Orthonormalization multigrid over the ranks of `group`.  `hierarchy`
    is the same global hierarchy object on every rank (ours or the
    reference's); b: the global level-1 right-hand side (numpy).  Returns
    (x_local numpy, (r0, r1) level-1 block rows, SolverReport)."""
    from .blockmatrix import as_block_sparse
    from .schwarz import schwarz_partition

    ctx = Context.get()
    comm = Comm(group)
    dev = ctx.device
    t_start = perf_counter()
    nl = hierarchy.num_levels
    k_lo = config.k_lo_scalar
    L = []
    for lam in range(1, nl + 1):
        lv = hierarchy.level(lam)
        config.check_degree(lv.data.basis.degree)
        rp, col, val = as_block_sparse(lv.matrix).bsr_arrays()
        N = val.shape[1]
        nb = len(rp) - 1
        P = balanced_row_starts(nb, comm.world)
        d = dict(N=N, P=P, r0=int(P[comm.rank]), r1=int(P[comm.rank + 1]))
        coarsest = lam == nl or lv.restriction is None
        if coarsest:
            Dc = DeviceBSR.from_arrays(rp, col, val, N, nb, ctx)
            d["direct"] = (SparseDirect(Dc, ctx) if nb * N > SPARSE_DIRECT_MIN
                           else DeviceDirect(dense_from_device_bsr(Dc), ctx))
            d["counts"] = [int(P[q + 1] - P[q]) * N for q in range(comm.world)]
            d["coarsest"] = True
            L.append(d)
            break
        d["coarsest"] = False
        d["M"] = _DistOp(local_operator(rp, col, val, N, P, comm.rank, ctx), P, comm, ctx, group)
        target = max(config.schwarz_target_dofs, lv.data.block_size)
        part = schwarz_partition(lv.graph, lv.data, target)
        m = min(space_dimension(k_lo, part.dim), N)
        d["S"] = _DistSchwarz(rp, col, val, N, part, m, P, comm, ctx, group)
        R = as_block_sparse(lv.restriction)
        Rrp, Rcol, Rval = R.bsr_arrays()
        ncoarse = R.col_layout.num_blocks
        Pc = balanced_row_starts(ncoarse, comm.world)
        d["R"] = _DistOp(local_rect_operator(Rrp, Rcol, Rval, N, P, Pc, comm.rank, ctx),
                         Pc, comm, ctx, group)
        Trp, Tcol, Tval = _transpose_bsr(Rrp, Rcol, Rval, ncoarse)
        d["Rt"] = _DistOp(local_rect_operator(Trp, Tcol, Tval, N, Pc, P, comm.rank, ctx),
                          P, comm, ctx, group)
        n = (d["r1"] - d["r0"]) * N
        d["rm"] = _DistRm(n, config.rm_max_columns, d["M"], comm, ctx)
        d["z"] = torch.zeros(n, dtype=F64, device=dev)
        d["xf"] = torch.zeros(n, dtype=F64, device=dev)
        L.append(d)
    for i in range(len(L) - 1):
        d = L[i + 1]
        n = (d["r1"] - d["r0"]) * d["N"]
        d["b"] = torch.zeros(n, dtype=F64, device=dev)
        d["xc"] = torch.zeros(n, dtype=F64, device=dev)

    def level(i, bl, xout, budget, hist):
        d = L[i]
        if d["coarsest"]:
            bfull = comm.allgather_cat(bl, d["counts"])
            xfull = d["direct"].apply(bfull)
            xout.copy_(xfull[d["r0"] * d["N"]: d["r1"] * d["N"]])
            if hist is not None:
                raise NotImplementedError("single-level hierarchy: use direct_factor")
            return 0
        rm, M, S = d["rm"], d["M"], d["S"]
        r = torch.empty_like(bl)
        M(xout, r)
        ctx.sub(bl, r, r)
        rm.init(xout, r)
        if hist is not None:
            hist.append(rm.best)
        it = 0
        while rm.best > config.tolerance and it < budget:
            it += 1
            S(rm.r, d["z"])
            rm.step(d["z"])
            nxt = L[i + 1]
            d["Rt"](rm.r, nxt["b"])
            nxt["xc"].zero_()
            level(i + 1, nxt["b"], nxt["xc"], config.coarse_cycle_iterations, None)
            d["R"](nxt["xc"], d["xf"])
            rm.step(d["xf"])
            S(rm.r, d["z"])
            rm.step(d["z"])
            if hist is not None:
                hist.append(rm.best)
        if it > 0:
            xout.copy_(rm.x)
        return it

    d0 = L[0]
    bl = torch.from_numpy(np.ascontiguousarray(
        b[d0["r0"] * d0["N"]: d0["r1"] * d0["N"]], float)).to(dev)
    x = torch.zeros_like(bl)
    hist: list = []
    it = level(0, bl, x, config.max_iterations, hist)
    torch.cuda.synchronize(dev)
    rep = SolverReport(solver="omg", iterations=it, converged=hist[-1] <= config.tolerance,
                       final_residual=hist[-1], residual_history=hist,
                       time_iterations=perf_counter() - t_start,
                       dofs=(len(as_block_sparse(hierarchy.level(1).matrix).bsr_arrays()[0]) - 1)
                       * d0["N"])
    return x.cpu().numpy(), (d0["r0"], d0["r1"]), rep
