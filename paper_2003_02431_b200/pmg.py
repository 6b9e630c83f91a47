"""Device plan for the degree-separated block preconditioner over a batch of
cell sets (cutdg solvers.py:183-305) -- one set for `pmg_apply`/GMRES, all
extended Schwarz blocks of a partition for `schwarz_apply`
(solvers.py:460-478).

Setup (counted in the solve time, like the reference's lazy factorisations,
solvers.py:300-305):
  * per set S: restricted block lists (extract_block_submatrix semantics),
    dense low-order matrix A_S (modes < m of every block in S x S) built on
    the device, pivoted LU;
  * per cell: pivoted LU of the high-order diagonal block H_c, shared by
    every set containing the cell (H_c depends only on M[c, c]).
Apply (3 launches, all sets at once):
  xdg_lu_inv_apply_*    -> x_lo of every set (triangular-inverse GEMVs)
  xdg_pmg_high          -> residual on the high rows + per-cell H_c solves
  xdg_pmg_combine       -> ordered sum over sets / damping (or scatter)
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .factor import batched_factor, buckets_by_size
from .errors import SingularSystemError

F64 = torch.float64
I32 = torch.int32
I64 = torch.int64


def _ranges(starts: np.ndarray, ends: np.ndarray) -> np.ndarray:
    """Concatenation of arange(s, e) for each pair (vectorised)."""
    lens = ends - starts
    if lens.sum() == 0:
        return np.zeros(0, np.int64)
    offs = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return np.arange(lens.sum(), dtype=np.int64) + offs


# Low-order factor selection.  A dense solve streams 8 n^2 bytes in 3
# launches; the multifrontal one ~8 (p^2 + 2 p b) per front in 2 launches per
# tree height and sweep.  For the 336,610-unknown global system of GMRES-PMG
# dense is impossible (906 GB).  For Schwarz plans the multifrontal factors
# move fewer bytes per application but cost more setup (host symbolic phase,
# hundreds of front buckets), so they pay off when the plan's dense factors
# are large.  Measured on B200 (round 2 session 5, OMG cold solves incl. the
# lazy setup, `profiles/r2_omg_loworder_full.txt`): cfg2 level 1 (337
# systems of ~1,810 unknowns, 8.8 GB dense) 15.1 s dense vs 14.2 s sparse
# (steady-state 13.8 vs 10.9 s); 16^3 p=3 (1.7 GB dense) 4.13 vs 4.02 s;
# 8^3 p=3 (0.2 GB) 1.47 vs 1.66 s; cfg4 at 16^3 0.54 vs 1.37 s.  Sparse when
# a system is larger than DENSE_LOW_MAX_SYSTEM unknowns, when the plan's
# dense factors exceed SPARSE_MIN_DENSE_BYTES, or when they would take more
# than 0.6 of the free device memory.
DENSE_LOW_MAX_SYSTEM = 16000  # unknowns
SPARSE_MIN_DENSE_BYTES = 1.0e9
# dense solves by CTA tasks with the right-hand side in shared memory: when
# there are enough tasks to fill the GPU (4 CTAs per SM) and each system fits
# 48 KB.  Measured at cfg2 level 1 (337 systems of ~1,810 unknowns): 5.0 TB/s
# vs 4.2 TB/s for the per-row kernel.
TASK_MIN_TASKS = 8 * 148
TASK_MAX_DIM = 6144
ROWS_PER_TASK = 32  # measured: 32 / 64 / 128 / 256 rows -> cfg2 OMG 17.29 / 17.47 / 17.79 / 18.81 s


def use_multifrontal(dims) -> bool:
    import os

    mode = os.environ.get("XDG_LOW_ORDER", "auto")
    if mode in ("dense", "sparse"):
        return mode == "sparse"
    dims = np.asarray(dims, np.int64)
    if dims.size == 0:
        return False
    free, _ = torch.cuda.mem_get_info()
    # the dense factors are built in place and factored in <= 2 GB chunks
    dense_bytes = 8 * int((dims * dims).sum())
    return (int(dims.max()) > DENSE_LOW_MAX_SYSTEM or dense_bytes > SPARSE_MIN_DENSE_BYTES
            or dense_bytes > 0.6 * free)


class PmgPlan:
    def __init__(self, D, cell_sets, m: int, damping: torch.Tensor | None = None,
                 combine: bool = True):
        """D: DeviceBSR (square, uniform N); cell_sets: list of sorted int
        arrays; m: number of low modes (1 <= m <= N)."""
        ctx = D.ctx
        self.ctx, self.D, self.m = ctx, D, int(m)
        N = D.N
        self.N = N
        dev = ctx.device
        rp = D.row_ptr.cpu().numpy().astype(np.int64)
        col = D.col.cpu().numpy().astype(np.int64)
        nbr = D.nbr
        self.nsys = len(cell_sets)
        sets = [np.asarray(S, np.int64) for S in cell_sets]
        self.sets = sets

        # ---- restricted block lists per work item (set, local row) -------
        loc = np.full(nbr, -1, np.int64)
        wi_cnt, wi_blk, wi_lcol, wi_cell, wi_lrow, wi_sys = [], [], [], [], [], []
        for s, S in enumerate(sets):
            loc[S] = np.arange(len(S))
            ks = _ranges(rp[S], rp[S + 1])
            lc = loc[col[ks]]
            keep = lc >= 0
            rows = np.repeat(np.arange(len(S)), rp[S + 1] - rp[S])
            wi_cnt.append(np.bincount(rows[keep], minlength=len(S)))
            wi_blk.append(ks[keep])
            wi_lcol.append(lc[keep])
            wi_cell.append(S)
            wi_lrow.append(np.arange(len(S)))
            wi_sys.append(np.full(len(S), s))
            loc[S] = -1
        cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64))
        cnt = cat(wi_cnt)
        self.nwork = len(cnt)
        wi_ptr = np.zeros(self.nwork + 1, np.int64)
        np.cumsum(cnt, out=wi_ptr[1:])
        wcell, wlrow, wsys = cat(wi_cell), cat(wi_lrow), cat(wi_sys)

        sizes = np.array([len(S) for S in sets], np.int64)
        dims = sizes * self.m
        vec_off = np.zeros(self.nsys + 1, np.int64)
        np.cumsum(dims, out=vec_off[1:])
        lu_off = np.zeros(self.nsys + 1, np.int64)
        np.cumsum(dims * dims, out=lu_off[1:])
        out_off = np.zeros(self.nsys + 1, np.int64)
        np.cumsum(sizes * N, out=out_off[1:])

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)

        self.wi_ptr = up(wi_ptr, I32)
        self.wi_blk = up(cat(wi_blk), I32)
        self.wi_lcol = up(cat(wi_lcol), I32)
        self.wi_cell = up(wcell, I32)
        self.wi_lrow = up(wlrow, I32)
        self.wi_sys = up(wsys, I32)
        self.dims = up(dims, I32)
        self.vec_off = up(vec_off[:-1], I64)
        self.lu_off = up(lu_off[:-1], I64)
        self.xlo = torch.zeros(int(vec_off[-1]), dtype=F64, device=dev)

        self.total = int(vec_off[-1])
        self.mf = None
        self.task_sys = None
        if use_multifrontal(dims):
            # ---- low-order sparse factors (solvers.py:208-221) -----------
            from .multifrontal import Multifrontal

            vsrc = np.concatenate(sets) * N if sets else np.zeros(0, np.int64)
            vdst = vec_off[:-1][wsys] + wlrow * self.m
            self.mf = Multifrontal(ctx, rp, col, D.val_t, N, sets, self.m, vsrc, vdst,
                                   what="low-order system")
            self.LU = torch.zeros(1, dtype=F64, device=dev)
            self.src = torch.zeros(1, dtype=I32, device=dev)
            self.row_sys = torch.zeros(1, dtype=I32, device=dev)
            self.lu_scratch = torch.zeros(2, dtype=F64, device=dev)
        else:
            self._dense_low(ctx, D, sets, dims, vec_off, lu_off, up)
        self._high_and_out(ctx, D, rp, col, nbr, sets, wcell, wlrow, wsys, vec_off,
                           out_off, combine, damping, up)

    def _dense_low(self, ctx, D, sets, dims, vec_off, lu_off, up):
        N, dev = self.N, ctx.device
        # ---- low-order dense factors (solvers.py:208-221) ----------------
        need = 8 * int(lu_off[-1])
        free, _ = torch.cuda.mem_get_info(dev)
        if need + (3 << 30) > free:  # factors (in place) + the <= 2 GB sweep workspace
            raise NotImplementedError(
                f"dense low-order factors need {need / 1e9:.1f} GB (largest system "
                f"{int(dims.max())} unknowns; {free / 1e9:.0f} GB free): use the "
                "multifrontal factorization (XDG_LOW_ORDER=auto|sparse)")
        A = torch.zeros(int(lu_off[-1]), dtype=F64, device=dev)
        nat.check(ctx.lib.xdg_pmg_build_low(
            self.nwork, N, self.m, self.wi_ptr.data_ptr(),
            self.wi_blk.data_ptr(), self.wi_lcol.data_ptr(),
            self.wi_lrow.data_ptr(), self.wi_sys.data_ptr(),
            self.lu_off.data_ptr(), self.dims.data_ptr(), D.val_t.data_ptr(),
            A.data_ptr(), ctx.stream), "pmg_build_low")
        # factor every system in place (xdg_batched_factor: partial-pivoting
        # LU, then the triangular inverses the solve kernels read), one call
        # per size bucket; permutations land at the systems' vector offsets.
        # One deferred singularity check for all systems.
        perm = torch.zeros(max(int(vec_off[-1]), 1), dtype=I32, device=dev)
        infos = []
        for idx in buckets_by_size(dims):
            idx = idx[dims[idx] > 0]
            if not len(idx):
                continue
            _, _, info = batched_factor(ctx, A, lu_off[idx], dims[idx], invert=True,
                                        perm=perm, perm_off=vec_off[idx])
            infos.append((idx, info[:len(idx)]))
        for idx, info in infos:
            bad = torch.nonzero(info)
            if bad.numel():
                cells = tuple(int(c) for c in sets[int(idx[int(bad[0])])][:8])
                raise SingularSystemError(f"low-order system on cells {cells}... is singular")
        self.LU = A
        perm = perm[:int(vec_off[-1])].long()
        # src = global DOF of local low unknown perm[i]:  cell*N + mode
        gidx = torch.from_numpy(
            np.concatenate([np.repeat(S * N, self.m) + np.tile(np.arange(self.m), len(S))
                            for S in sets]) if sets else np.zeros(0, np.int64)).to(dev)
        base = torch.from_numpy(np.repeat(vec_off[:-1], dims)).to(dev)
        # perm is local to each system: global position = base + local index
        self.src = gidx[base + perm].to(I32) if perm.numel() else perm.to(I32)
        # packed-row -> system map for the warp-per-row inverse apply
        self.row_sys = up(np.repeat(np.arange(self.nsys), dims), I32)
        self.lu_scratch = torch.empty(2 * max(self.total, 1), dtype=F64, device=dev)
        # CTA tasks (system, 64-row block) with the right-hand side staged in
        # shared memory (xdg_lu_inv_apply_tasks): many systems that fit
        nblk = (dims + ROWS_PER_TASK - 1) // ROWS_PER_TASK
        if int(nblk.sum()) >= TASK_MIN_TASKS and 0 < int(dims.max()) <= TASK_MAX_DIM:
            self.task_sys = up(np.repeat(np.arange(self.nsys), nblk), I32)
            self.task_row0 = up(_ranges(np.zeros(self.nsys, np.int64), nblk) * ROWS_PER_TASK,
                                I32)
            self.rows_per_task, self.max_dim = ROWS_PER_TASK, int(dims.max())

    def _high_and_out(self, ctx, D, rp, col, nbr, sets, wcell, wlrow, wsys, vec_off,
                      out_off, combine, damping, up):
        N, dev = self.N, ctx.device
        # ---- high-order per-cell factors (solvers.py:225-243) ------------
        self.has_high = self.m < N
        if self.has_high:
            nh = N - self.m
            ucells = np.unique(wcell) if len(wcell) else np.zeros(0, np.int64)
            rows_of_k = np.repeat(np.arange(nbr), rp[1:] - rp[:-1])
            diag_k = np.full(nbr, -1, np.int64)
            isdiag = col == rows_of_k
            diag_k[rows_of_k[isdiag]] = np.flatnonzero(isdiag)
            missing = ucells[diag_k[ucells] < 0]
            if len(missing):
                raise SingularSystemError(f"cell {int(missing[0])} has no diagonal block")
            H = torch.empty(len(ucells) * nh * nh, dtype=F64, device=dev)
            nat.check(ctx.lib.xdg_pmg_gather_high(
                len(ucells), N, self.m, up(ucells, I32).data_ptr(),
                up(diag_k[ucells], I32).data_ptr(), D.val_t.data_ptr(),
                H.data_ptr(), ctx.stream), "pmg_gather_high")
            # per-cell partial-pivoting LU in place (xdg_batched_factor; the
            # reference's scipy lu_factor, solvers.py:233), column-major copy
            # for the warp-per-cell solve
            nu = len(ucells)
            hoff = np.arange(nu, dtype=np.int64) * nh
            hperm, _, info = batched_factor(ctx, H, hoff * nh, np.full(nu, nh, np.int32),
                                            invert=False, perm_off=hoff)
            bad = torch.nonzero(info[:nu])
            if bad.numel():
                c = int(ucells[int(bad[0])])
                raise SingularSystemError(f"high-order block of cell {c} is singular")
            self.HLU = torch.empty_like(H)
            nat.check(ctx.lib.xdg_blocks_transpose(
                nu, nh, H.data_ptr(), self.HLU.data_ptr(), ctx.stream), "blocks_transpose(H)")
            self.hperm = hperm
            hidx = np.full(nbr, -1, np.int64)
            hidx[ucells] = np.arange(len(ucells))
            self.wi_hidx = up(hidx[wcell], I32)
            self.wi_xlo = up(vec_off[:-1][wsys], I64)

        # ---- output placement ---------------------------------------------
        # direct mode: one set equal to all rows in order -> write z in place
        self.direct = (not combine and self.nsys == 1 and len(sets[0]) == nbr
                       and np.array_equal(sets[0], np.arange(nbr)))
        if self.direct:
            self.wi_out = up(wcell * N, I64) if self.has_high else None
            self.out = None
        else:
            self.wi_out = up(out_off[:-1][wsys] + wlrow * N, I64)
            # out buffer: the low-only case reuses xlo (same local layout)
            self.out = (torch.empty(int(out_off[-1]), dtype=F64, device=dev)
                        if self.has_high else self.xlo)
            order = np.lexsort((wsys, wcell))  # by cell, then set index
            cptr = np.zeros(nbr + 1, np.int64)
            np.cumsum(np.bincount(wcell, minlength=nbr), out=cptr[1:])
            cpos = (out_off[:-1][wsys] + wlrow * N)[order]
            self.cptr = up(cptr, I32)
            self.cpos = up(cpos, I64)
        self.damping = damping

    # ------------------------------------------------------------------
    def apply(self, b: torch.Tensor, z: torch.Tensor) -> torch.Tensor:
        """z = sum_S PMG_S(b) ./ damping   (or the single-set PMG), through
        the native xdg_pmg_apply_op."""
        import ctypes as C

        from .driver import bsr_struct, pmg_struct

        if getattr(self, "_struct", None) is None:
            self._struct = pmg_struct(self)
        Ms = bsr_struct(self.D)
        nat.check(self.ctx.lib.xdg_pmg_apply_op(
            C.byref(self._struct[0]), C.byref(Ms), b.data_ptr(), z.data_ptr(),
            self.ctx.stream), "pmg_apply")
        return z

    def algorithmic_bytes(self) -> int:
        """Bytes one apply must move (SURVEY 8(d) PMG apply)."""
        N, m = self.N, self.m
        lo = (self.mf.apply_bytes if self.mf is not None
              else int(self.dims.double().pow(2).sum().item()) * 8)
        hi = 0
        if self.has_high:
            nh = N - m
            hi = self.nwork * nh * nh * 8 + int(self.wi_blk.numel()) * (nh * m * 8 + 4)
        vec = self.nwork * N * 8 * 3
        return lo + hi + vec
