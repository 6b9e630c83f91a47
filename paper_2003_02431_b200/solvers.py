"""Drop-in `cutdg.solvers` (reference: /root/reference/pkg/src/cutdg/solvers.py)
running on the B200.

Same public names, signatures, defaults, error classes and report
semantics as the reference.  Python builds the device plans (setup, counted
inside `time_iterations` like the reference's lazy factorisations); the
iteration loops run in the native C++ driver of libxdg_b200.so, which makes
the reference's scalar decisions (dependent candidate, accept/reject,
Givens, convergence) on the host and launches every vector operation as a
kernel:

  pmg_apply / schwarz_apply   -> pmg.PmgPlan -> xdg_pmg_apply_op (triangular-
                                 inverse LU applies + fused high-order
                                 residual/solve + ordered combine)
  rm_step / RmState           -> xdg_rm_step (SpMV with fused norm, W^T w /
                                 W c kernels, fused exact-image update; one
                                 host sync per step)
  ortho_mg_solve              -> xdg_omg_solve (recursion over the level
                                 structs; R, R^T products are BSR SpMVs)
  gmres_pmg_solve             -> xdg_gmres_solve (cooperative fused MGS, one
                                 host sync per inner iteration)

Public functions accept numpy arrays (returning numpy, like the reference)
or CUDA tensors (returning CUDA tensors, zero-copy for device callers).
"""
from __future__ import annotations

import csv
import ctypes as C
import math
from dataclasses import dataclass
from math import comb
from time import perf_counter
from typing import Optional, Sequence

import numpy as np
import torch

from .blockmatrix import as_block_sparse
from .device import Context, DeviceBSR
from .direct import DirectFactorization, direct_factor
from .driver import RmBuffers, XdgOmgLevel, bsr_struct, direct_struct, pmg_struct
from ._native import check as nat_check
from .errors import (
    DimensionMismatchError,
    InvalidConfigError,
    LayoutMismatchError,
)
from .pmg import PmgPlan
from .schwarz import SchwarzPartition, schwarz_partition

__all__ = [
    "DEPENDENT_CANDIDATE_RTOL", "DEFAULT_RM_MAX_COLUMNS", "SolverConfig",
    "SolverReport", "REPORT_CSV_HEADER", "pmg_apply", "SchwarzPartition",
    "schwarz_partition", "schwarz_apply", "RmState", "rm_step",
    "ortho_mg_solve", "gmres_pmg_solve", "space_dimension",
]

DEPENDENT_CANDIDATE_RTOL = 1e-13   # solvers.py:52
LAST_LOOP: dict = {}               # last GMRES loop: seconds, algorithmic bytes
DEFAULT_RM_MAX_COLUMNS = 200       # solvers.py:53
F64 = torch.float64


def space_dimension(degree: int, dim: int) -> int:
    """N_k = binomial(k + D, D) (basis.py:29-31)."""
    return comb(degree + dim, dim)


# ---------------------------------------------------------------------------
# configuration and reporting (solvers.py:60-152)


@dataclass(frozen=True)
class SolverConfig:
    tolerance: float = 1e-10
    max_iterations: int = 1000
    k_lo: tuple = (1,)
    schwarz_target_dofs: int = 2000
    gmres_restart: int = 30
    num_levels: int = 2
    rm_max_columns: int = DEFAULT_RM_MAX_COLUMNS
    coarse_cycle_iterations: int = 2

    def __post_init__(self):
        if not self.tolerance > 0:
            raise InvalidConfigError("tolerance must be positive")
        if self.max_iterations < 0:
            raise InvalidConfigError("max_iterations must be >= 0")
        k = self.k_lo
        if isinstance(k, tuple):
            klo = k
        elif isinstance(k, (list, np.ndarray)):
            klo = tuple(k)
        else:
            klo = (k,)
        object.__setattr__(self, "k_lo", klo)
        if any(int(v) < 0 for v in klo):
            raise InvalidConfigError("k_lo entries must be >= 0")
        if self.gmres_restart < 1:
            raise InvalidConfigError("gmres_restart must be >= 1")
        if self.num_levels < 1:
            raise InvalidConfigError("num_levels must be >= 1")
        if self.rm_max_columns < 1:
            raise InvalidConfigError("rm_max_columns must be >= 1")
        if self.coarse_cycle_iterations < 1:
            raise InvalidConfigError("coarse_cycle_iterations must be >= 1")

    @property
    def k_lo_scalar(self) -> int:
        return int(self.k_lo[0])

    def check_degree(self, k: int) -> None:
        if any(int(v) > k for v in self.k_lo):
            raise InvalidConfigError(f"k_lo {self.k_lo} exceeds the space degree {k}")


REPORT_CSV_HEADER = (
    "solver,dofs,iterations,converged,setup_basis_ms,"
    "setup_matmat_ms,solve_ms,final_residual"
)


@dataclass
class SolverReport:
    solver: str
    iterations: int
    converged: bool
    final_residual: float
    residual_history: list
    time_basis_setup: float = 0.0
    time_matmat_setup: float = 0.0
    time_iterations: float = 0.0
    dofs: int = 0

    def csv_row(self) -> str:
        return ",".join([
            self.solver, str(self.dofs), str(self.iterations),
            str(self.converged).lower(),
            f"{1e3 * self.time_basis_setup:.3f}",
            f"{1e3 * self.time_matmat_setup:.3f}",
            f"{1e3 * self.time_iterations:.3f}",
            f"{self.final_residual:.6e}",
        ])

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            fh.write(REPORT_CSV_HEADER + "\n" + self.csv_row() + "\n")

    def write_history_csv(self, path) -> None:
        with open(path, "w", newline="") as fh:
            out = csv.writer(fh)
            out.writerow(["iteration", "residual"])
            for i, r in enumerate(self.residual_history):
                out.writerow([i, f"{r:.16e}"])


# ---------------------------------------------------------------------------
# host <-> device helpers


def _is_dev(v) -> bool:
    return torch.is_tensor(v) and v.is_cuda


def _to_dev(v, ctx: Context, copy: bool = True) -> torch.Tensor:
    if torch.is_tensor(v):
        t = v.to(device=ctx.device, dtype=F64)
        if copy and t.data_ptr() == v.data_ptr():
            t = t.clone()
        return t.contiguous()
    return torch.from_numpy(np.array(v, dtype=float, copy=True)).to(ctx.device)


def _out(t: torch.Tensor, like_dev: bool):
    return t if like_dev else t.cpu().numpy()


def _length(v) -> tuple:
    return tuple(v.shape) if (torch.is_tensor(v) or isinstance(v, np.ndarray)) \
        else np.asarray(v).shape


def _device_operator(M, ctx: Context) -> DeviceBSR:
    """Device mirror of anything the reference's solvers accept as M: a
    BlockSparseMatrix (ours or the reference's), a DeviceBSR, or a dense
    array (rm_step's `M @ v` branch, solvers.py:581-584)."""
    if isinstance(M, DeviceBSR):
        return M
    if hasattr(M, "blocks") and hasattr(M, "row_layout"):
        return as_block_sparse(M).device(ctx)
    A = np.asarray(M, dtype=float)
    if A.ndim != 2 or A.shape[0] != A.shape[1]:
        raise DimensionMismatchError("operator must be square")
    n = A.shape[0]
    return DeviceBSR.from_arrays(np.array([0, 1]), np.array([0]),
                                 A.reshape(1, n, n), n, 1, ctx)


# ---------------------------------------------------------------------------
# degree-separated block preconditioner (solvers.py:159-305)


def _normalize_k_lo(k_lo) -> int:
    if isinstance(k_lo, (int, np.integer)):
        val = int(k_lo)
    else:
        seq = tuple(k_lo)
        if len(seq) != 1:
            raise InvalidConfigError("one separation degree expected for a scalar unknown")
        val = int(seq[0])
    if val < 0:
        raise InvalidConfigError("separation degree must be >= 0")
    return val


def _uniform_block_size(M) -> int:
    sizes = set(M.row_layout.sizes) | set(M.col_layout.sizes)
    if len(sizes) != 1:
        raise LayoutMismatchError(
            "degree-separated preconditioning needs a uniform block layout")
    return sizes.pop()


def _pmg_plan(M, D: DeviceBSR, cells: tuple, modes_low: int, cache: dict) -> PmgPlan:
    key = (cells, modes_low)
    plan = cache.get(key)
    if plan is None:
        plan = PmgPlan(D, [np.asarray(cells, np.int64)], modes_low, combine=False)
        cache[key] = plan
    return plan


def pmg_apply(M, b, k_lo, cells: Sequence[int], factorization_cache: dict, *,
              dim: int):
    """One application of the degree-separated preconditioner on the block
    rows `cells` (solvers.py:268-305); output supported on `cells` only;
    factorizations cached in `factorization_cache` keyed (cells, modes)."""
    klo = _normalize_k_lo(k_lo)
    block_size = _uniform_block_size(M)
    modes_low = min(space_dimension(klo, dim), block_size)
    cells = tuple(sorted(set(int(c) for c in cells)))
    if not cells:
        raise InvalidConfigError("empty cell set")
    if cells[0] < 0 or cells[-1] >= M.row_layout.num_blocks:
        raise DimensionMismatchError("cell index out of range")
    if _length(b) != (M.shape[0],):
        raise DimensionMismatchError(f"rhs of length {_length(b)} against matrix {M.shape}")
    ctx = Context.get()
    D = _device_operator(M, ctx)
    plan = _pmg_plan(M, D, cells, modes_low, factorization_cache)
    bd = _to_dev(b, ctx, copy=False)
    z = torch.zeros(M.shape[0], dtype=F64, device=ctx.device)
    plan.apply(bd, z)
    return _out(z, _is_dev(b))


# ---------------------------------------------------------------------------
# additive overlapping-block smoother (solvers.py:460-478)


def _schwarz_plan(M, D: DeviceBSR, partition: SchwarzPartition, modes_low: int,
                  ctx: Context) -> PmgPlan:
    key = ("__xdg_schwarz__", modes_low)
    plan = partition.cache.get(key)
    if plan is None:
        damp = torch.from_numpy(np.asarray(partition.damping, float)).to(ctx.device)
        plan = PmgPlan(D, [np.asarray(r, np.int64) for r in partition.block_rows],
                       modes_low, damping=damp, combine=True)
        partition.cache[key] = plan
    return plan


def _schwarz_dev(M, D, r: torch.Tensor, partition, k_lo, ctx, z=None):
    klo = _normalize_k_lo(k_lo)
    modes_low = min(space_dimension(klo, partition.dim), _uniform_block_size(M))
    plan = _schwarz_plan(M, D, partition, modes_low, ctx)
    if z is None:
        z = torch.empty_like(r)
    return plan.apply(r, z)


def schwarz_apply(M, residual, partition: SchwarzPartition, k_lo):
    """z = (sum over extended blocks of PMG_block(residual)) ./ damping."""
    if _length(residual) != (M.shape[0],):
        raise DimensionMismatchError(
            f"residual of length {_length(residual)} against matrix {M.shape}")
    if len(partition.damping) != M.shape[0]:
        raise DimensionMismatchError("partition built for another layout")
    for rows in partition.block_rows:
        if not rows:
            raise InvalidConfigError("empty cell set")
    ctx = Context.get()
    D = _device_operator(M, ctx)
    z = _schwarz_dev(M, D, _to_dev(residual, ctx, copy=False), partition, k_lo, ctx)
    return _out(z, _is_dev(residual))


# ---------------------------------------------------------------------------
# residual minimization (solvers.py:485-625) -- native driver (xdg_rm_*)


class RmState:
    """Growing orthonormal search space (solvers.py:485-556), device
    resident: W, Z are (max_columns, L) buffers in HBM, counters live in the
    native `xdg_rm` struct that xdg_rm_step updates.  `W`, `Z`, `alpha`,
    `x0`, `r0`, `current()` return host copies for inspection."""

    def __init__(self, x0, r0, max_columns: int = DEFAULT_RM_MAX_COLUMNS):
        if _length(x0) != _length(r0):
            raise DimensionMismatchError("x0 and r0 lengths differ")
        if max_columns < 1:
            raise InvalidConfigError("max_columns must be >= 1")
        ctx = Context.get()
        self._ctx = ctx
        xd, rd = _to_dev(x0, ctx), _to_dev(r0, ctx)
        self.n = xd.numel()
        self.max_columns = int(max_columns)
        self._buf = RmBuffers(ctx, self.n, self.max_columns)
        nat_check(ctx.lib.xdg_rm_init(C.byref(self._buf.s), xd.data_ptr(),
                                      rd.data_ptr(), ctx.stream), "rm_init")

    # counters / scalars of the native state (reference attribute names)
    ncols = property(lambda self: self._buf.s.ncols)
    best_norm = property(lambda self: self._buf.s.best_norm)
    last_dependent = property(lambda self: bool(self._buf.s.last_dependent))
    dependent_count = property(lambda self: self._buf.s.dependent_count)
    rejected_count = property(lambda self: self._buf.s.rejected_count)
    restart_count = property(lambda self: self._buf.s.restart_count)

    @property
    def x0(self):
        return self._buf.x0.cpu().numpy()

    @property
    def r0(self):
        return self._buf.r0.cpu().numpy()

    @property
    def W(self):
        return self._buf.W[: self.ncols].T.cpu().numpy()

    @property
    def Z(self):
        return self._buf.Z[: self.ncols].T.cpu().numpy()

    @property
    def alpha(self):
        return self._buf.alpha_host[: self.ncols].copy()

    def current_dev(self) -> tuple:
        nat_check(self._ctx.lib.xdg_rm_current(C.byref(self._buf.s), self._ctx.stream),
                  "rm_current")
        return self._buf.x.clone(), self._buf.r.clone()

    def current(self) -> tuple:
        x, r = self.current_dev()
        return x.cpu().numpy(), r.cpu().numpy()

    def restart(self) -> None:
        """Collapse the space onto the current point (solvers.py:548-556)."""
        nat_check(self._ctx.lib.xdg_rm_restart(C.byref(self._buf.s), self._ctx.stream),
                  "rm_restart")


def rm_step(state: RmState, z_candidate, M) -> tuple:
    """Extend the search space by one candidate; returns (x, r, state) with
    the true residual of the new best point (solvers.py:559-625)."""
    if _length(z_candidate) != (state.n,):
        raise DimensionMismatchError("candidate length mismatch")
    ctx = state._ctx
    D = _device_operator(M, ctx)
    zd = _to_dev(z_candidate, ctx, copy=False)
    Ms = bsr_struct(D)
    nat_check(ctx.lib.xdg_rm_step(C.byref(state._buf.s), C.byref(Ms), zd.data_ptr(),
                                  ctx.stream), "rm_step")
    x, r = state._buf.x.clone(), state._buf.r.clone()
    host = not _is_dev(z_candidate)
    return _out(x, not host), _out(r, not host), state


# ---------------------------------------------------------------------------
# multigrid over the aggregation hierarchy (solvers.py:632-749)


class _OmgContext:
    """Per-solve caches (solvers.py:632-666) plus the native level structs."""

    def __init__(self, config: SolverConfig, entry_level: int = 1):
        self.config = config
        self.entry_level = entry_level
        self.partitions = {}
        self.transposes = {}
        self.coarse_factorization = {}
        self._dev = Context.get()
        self._native = None

    def partition(self, hierarchy, level: int) -> SchwarzPartition:
        part = self.partitions.get(level)
        if part is None:
            lv = hierarchy.level(level)
            target = max(self.config.schwarz_target_dofs, lv.data.block_size)
            part = schwarz_partition(lv.graph, lv.data, target)
            self.partitions[level] = part
        return part

    def restriction_transpose(self, hierarchy, level: int):
        Rt = self.transposes.get(level)
        if Rt is None:
            Rt = as_block_sparse(hierarchy.level(level).restriction).transpose()
            self.transposes[level] = Rt
        return Rt

    def coarse_solver(self, hierarchy, level: int) -> DirectFactorization:
        fact = self.coarse_factorization.get(level)
        if fact is None:
            fact = direct_factor(hierarchy.level(level).matrix)
            self.coarse_factorization[level] = fact
        return fact

    def native_levels(self, hierarchy, entry: int):
        """XdgOmgLevel array for levels entry..last visited (built once per
        hierarchy; a context reused at a lower entry level than the one the
        cached array was built for gets a rebuilt array -- the reference's
        context is valid for any level)."""
        got = self._native
        if got is not None and got[2] is hierarchy and got[3] <= entry:
            return got[0], got[1]
        ctx = self._dev
        cfg = self.config
        nl = hierarchy.num_levels
        arr = (XdgOmgLevel * nl)()
        keep = []
        k_lo = cfg.k_lo_scalar
        for lam in range(entry, nl + 1):
            lv = hierarchy.level(lam)
            cfg.check_degree(lv.data.basis.degree)
            M = as_block_sparse(lv.matrix)
            D = M.device(ctx)
            n = D.nbr * D.N
            L = arr[lam - 1]
            L.M = bsr_struct(D)
            coarsest = lam == nl or lv.restriction is None
            rm = RmBuffers(ctx, n, cfg.rm_max_columns, allocate_space=not coarsest)
            keep.append(rm)
            L.rm = rm.s
            bufs = torch.zeros(3, n, dtype=F64, device=ctx.device)
            keep.append(bufs)
            L.b, L.z, L.xf = (bufs[i].data_ptr() for i in range(3))
            if coarsest:
                dd = self.coarse_solver(hierarchy, lam)._dev
                L.direct, k = direct_struct(dd)
                keep += [dd, k]
                L.has_restriction = 0
                break
            part = self.partition(hierarchy, lam)
            modes_low = min(space_dimension(k_lo, part.dim), _uniform_block_size(M))
            plan = _schwarz_plan(M, D, part, modes_low, ctx)
            L.schwarz, k = pmg_struct(plan)
            keep += [plan, k]
            Rd = as_block_sparse(lv.restriction).device(ctx)
            Rtd = self.restriction_transpose(hierarchy, lam).device(ctx)
            L.R, L.Rt = bsr_struct(Rd), bsr_struct(Rtd)
            keep += [Rd, Rtd]
            L.has_restriction = 1
        self._native = (arr, keep, hierarchy, entry)
        return arr, keep


def ortho_mg_solve(hierarchy, b, x0=None, config: Optional[SolverConfig] = None,
                   level: int = 1, _context: Optional[_OmgContext] = None) -> tuple:
    """Orthonormalization multigrid (Alg. 4) on `level`; returns
    (solution, SolverReport); non-convergence is reported, not raised.
    The iteration loop runs in the native driver (xdg_omg_solve)."""
    config = config or SolverConfig()
    ctx_omg = _context or _OmgContext(config, entry_level=level)
    lv = hierarchy.level(level)
    if _length(b) != (lv.matrix.shape[0],):
        raise DimensionMismatchError(
            f"rhs of length {_length(b)} against matrix {lv.matrix.shape}")
    config.check_degree(lv.data.basis.degree)
    ctx = ctx_omg._dev
    bd = _to_dev(b, ctx)
    t_start = perf_counter()
    arr, _keep = ctx_omg.native_levels(hierarchy, level)
    n = bd.numel()
    x = torch.zeros_like(bd) if x0 is None else _to_dev(x0, ctx)
    hist = np.zeros(config.max_iterations + 2)
    it, hl, fin, nbytes = C.c_int(0), C.c_int(0), C.c_double(0.0), C.c_double(0.0)
    t_iter = perf_counter()
    nat_check(ctx.lib.xdg_omg_solve(
        arr, hierarchy.num_levels, level - 1, float(config.tolerance),
        int(config.max_iterations), int(config.coarse_cycle_iterations),
        bd.data_ptr(), x.data_ptr(), int(x0 is not None), C.byref(it),
        hist.ctypes.data, C.byref(hl), C.byref(fin), C.byref(nbytes), ctx.stream),
        "omg_solve")
    ctx_omg.last_loop = dict(seconds=perf_counter() - t_iter, bytes=nbytes.value,
                             setup_seconds=t_iter - t_start)
    history = [float(v) for v in hist[: hl.value]]
    rep = SolverReport(solver="omg", iterations=it.value,
                       converged=fin.value <= config.tolerance,
                       final_residual=fin.value, residual_history=history,
                       time_iterations=perf_counter() - t_start, dofs=n)
    return _out(x, _is_dev(b)), rep


# ---------------------------------------------------------------------------
# preconditioned GMRES (solvers.py:756-846)


def gmres_pmg_solve(M, b, config: Optional[SolverConfig] = None,
                    factorization_cache: Optional[dict] = None, *, dim: int,
                    x0=None) -> tuple:
    """Restarted GMRES, degree-separated preconditioner on the right, MGS
    orthogonalisation, Givens rotations; stops on the true residual.  The
    iteration loop runs in the native driver (xdg_gmres_solve)."""
    config = config or SolverConfig()
    cache = factorization_cache if factorization_cache is not None else {}
    if _length(b) != (M.shape[0],):
        raise DimensionMismatchError(f"rhs of length {_length(b)} against matrix {M.shape}")
    nb = M.row_layout.num_blocks
    all_cells = tuple(range(nb))
    m = config.gmres_restart
    ctx = Context.get()
    bd = _to_dev(b, ctx)
    t_start = perf_counter()
    D = _device_operator(M, ctx)
    modes_low = min(space_dimension(_normalize_k_lo(config.k_lo_scalar), dim),
                    _uniform_block_size(M))
    plan = _pmg_plan(M, D, all_cells, modes_low, cache)
    n = bd.numel()
    dev = ctx.device
    x = torch.zeros_like(bd) if x0 is None else _to_dev(x0, ctx)
    V = torch.empty(m + 1, n, dtype=F64, device=dev)
    Z = torch.empty(m, n, dtype=F64, device=dev)
    w = torch.empty(n, dtype=F64, device=dev)
    r = torch.empty(n, dtype=F64, device=dev)
    sc = torch.zeros(m + 8, dtype=F64, device=dev)
    ycoef = torch.zeros(m, dtype=F64, device=dev)
    ws = torch.zeros((int(ctx.lib.xdg_reduce_workspace_bytes()) + 7) // 8, dtype=F64,
                     device=dev)
    hist = np.zeros(config.max_iterations + 2)
    it, hl, fin, nbytes = C.c_int(0), C.c_int(0), C.c_double(0.0), C.c_double(0.0)
    Ms = bsr_struct(D)
    Ps, _k = pmg_struct(plan)
    t_iter = perf_counter()
    nat_check(ctx.lib.xdg_gmres_solve(
        C.byref(Ms), C.byref(Ps), m, float(config.tolerance), int(config.max_iterations),
        bd.data_ptr(), x.data_ptr(), int(x0 is not None), V.data_ptr(), Z.data_ptr(),
        w.data_ptr(), r.data_ptr(), sc.data_ptr(), ycoef.data_ptr(), ws.data_ptr(),
        None, C.byref(it), hist.ctypes.data, C.byref(hl), C.byref(fin), C.byref(nbytes),
        ctx.stream), "gmres_solve")
    torch.cuda.synchronize(dev)
    LAST_LOOP.update(seconds=perf_counter() - t_iter, bytes=nbytes.value,
                     setup_seconds=t_iter - t_start)
    history = [float(v) for v in hist[: hl.value]]
    rep = SolverReport(solver="gmres-pmg", iterations=it.value,
                       converged=fin.value <= config.tolerance, final_residual=fin.value,
                       residual_history=history,
                       time_iterations=perf_counter() - t_start, dofs=M.shape[0])
    return _out(x, _is_dev(b)), rep
