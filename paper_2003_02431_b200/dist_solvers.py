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
from dataclasses import dataclass
from time import perf_counter

import numpy as np
import torch
import torch.distributed as dist

from . import _native as nat
from .device import Context, DeviceBSR
from .direct import DeviceDirect, dense_from_device_bsr, ipiv_to_perm
from .distributed import DistributedSpMV, HaloPlan
from .errors import SingularSystemError
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
    set, solvers.py:800), distributed: replicated global low-order solve +
    rank-local high-order stage."""

    def __init__(self, rp, col, val, N, m, op: LocalOperator, row_starts, comm: Comm, ctx):
        self.ctx, self.comm, self.op = ctx, comm, op
        self.N, self.m = N, m
        dev = ctx.device
        nbr = len(rp) - 1
        nloc = op.r1 - op.r0
        self.nloc = nloc
        self.counts = [int(row_starts[q + 1] - row_starts[q]) * m for q in range(comm.world)]
        # replicated low-order factor from the global blocks' (:m, :m) parts
        lo_val = np.ascontiguousarray(np.asarray(val)[:, :m, :m])
        Dlo = DeviceBSR.from_arrays(rp, col, lo_val, m, nbr, ctx)
        A = dense_from_device_bsr(Dlo)
        try:
            self.low = DeviceDirect(A, ctx, "low-order system")
        except SingularSystemError as exc:
            raise SingularSystemError("low-order system is singular") from exc
        del A, Dlo
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
            LUh, pvh, _ = torch.linalg.lu_factor_ex(H.view(nloc, nh, nh))
            dg = torch.diagonal(LUh, dim1=-2, dim2=-1)
            bad = (~torch.isfinite(LUh).flatten(1).all(1)) | (dg == 0).any(1)
            if bool(bad.any()):
                c = op.r0 + int(torch.nonzero(bad)[0])
                raise SingularSystemError(f"high-order block of cell {c} is singular")
            self.HLU = torch.empty_like(H)
            nat.check(ctx.lib.xdg_blocks_transpose(nloc, nh, LUh.contiguous().data_ptr(),
                                                   self.HLU.data_ptr(), ctx.stream), "transpose")
            self.hperm = ipiv_to_perm(ctx, pvh.to(I32).contiguous(),
                                      torch.full((nloc,), nh, dtype=I32, device=dev),
                                      torch.arange(nloc, dtype=torch.int64, device=dev) * nh)
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
            for i in range(j + 1):                       # modified Gram-Schmidt
                gdot(V[i], w, sc[i:i + 1])
                ctx.axpy(-1.0, V[i], w, a_dev=sc[i:i + 1])
            gdot(w, w, sc[j + 1:j + 2])
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
