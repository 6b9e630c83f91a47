"""Drop-in `cutdg.solvers` (reference: /root/reference/pkg/src/cutdg/solvers.py)
running on the B200.

Same public names, signatures, defaults, error classes and report
semantics as the reference; host Python keeps the control flow (restarts,
accept/reject, Givens rotations -- scalar work) while every vector-sized
operation runs in libxdg_b200.so on device-resident data:

  pmg_apply / schwarz_apply   -> pmg.PmgPlan (batched LU solves + fused
                                 high-order residual/solve + ordered combine)
  rm_step / RmState           -> SpMV with fused norm, W^T w / W c kernels,
                                 fused exact-image update
  ortho_mg_solve              -> recursion over device level mirrors;
                                 R, R^T products are BSR SpMVs
  gmres_pmg_solve             -> MGS with device scalars, one host sync per
                                 inner iteration (the Hessenberg column)

Public functions accept numpy arrays (returning numpy, like the reference)
or CUDA tensors (returning CUDA tensors, zero-copy for device callers).
"""
from __future__ import annotations

import csv
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
from .errors import (
    DimensionMismatchError,
    InvalidConfigError,
    LayoutMismatchError,
    SingularSystemError,
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


def _sync_read(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy()


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
# residual minimization (solvers.py:485-625)


class RmState:
    """Growing orthonormal search space (solvers.py:485-556), device
    resident: W, Z are (max_columns, L) row-per-column buffers in HBM.
    `W`, `Z`, `alpha`, `x0`, `r0`, `current()` return host copies for
    inspection; the solvers use the `_dev` views."""

    def __init__(self, x0, r0, max_columns: int = DEFAULT_RM_MAX_COLUMNS):
        if _length(x0) != _length(r0):
            raise DimensionMismatchError("x0 and r0 lengths differ")
        if max_columns < 1:
            raise InvalidConfigError("max_columns must be >= 1")
        ctx = Context.get()
        self._ctx = ctx
        self._host = not (_is_dev(x0) or _is_dev(r0))
        self._x0 = _to_dev(x0, ctx)
        self._r0 = _to_dev(r0, ctx)
        n = self._x0.numel()
        self.n = n
        self.max_columns = int(max_columns)
        dev = ctx.device
        self._W = torch.empty(self.max_columns, n, dtype=F64, device=dev)
        self._Z = torch.empty(self.max_columns, n, dtype=F64, device=dev)
        self._alpha = np.zeros(self.max_columns)
        self._y = torch.zeros(n, dtype=F64, device=dev)
        self._My = torch.zeros(n, dtype=F64, device=dev)
        self._Mz = torch.empty(n, dtype=F64, device=dev)
        self._My_new = torch.empty(n, dtype=F64, device=dev)
        self._coeff = torch.zeros(self.max_columns, dtype=F64, device=dev)
        self._sc = torch.zeros(8, dtype=F64, device=dev)
        self.best_norm = self._norm(self._r0)
        self.ncols = 0
        self.last_dependent = False
        self.dependent_count = 0
        self.rejected_count = 0
        self.restart_count = 0

    def _norm(self, v: torch.Tensor) -> float:
        self._ctx.dot(v, v, self._sc[7:8])
        return math.sqrt(float(_sync_read(self._sc[7:8])[0]))

    # host views (reference attribute semantics)
    @property
    def x0(self):
        return self._x0.cpu().numpy()

    @property
    def r0(self):
        return self._r0.cpu().numpy()

    @property
    def W(self):
        return self._W[: self.ncols].T.cpu().numpy()

    @property
    def Z(self):
        return self._Z[: self.ncols].T.cpu().numpy()

    @property
    def alpha(self):
        return self._alpha[: self.ncols].copy()

    def current_dev(self) -> tuple:
        ctx = self._ctx
        x = torch.empty_like(self._x0)
        r = torch.empty_like(self._r0)
        ctx.lib.xdg_add(self.n, self._x0.data_ptr(), self._y.data_ptr(),
                        x.data_ptr(), ctx.stream)
        ctx.sub(self._r0, self._My, r)
        return x, r

    def current(self) -> tuple:
        x, r = self.current_dev()
        return x.cpu().numpy(), r.cpu().numpy()

    def restart(self) -> None:
        """Collapse the space onto the current point (solvers.py:548-556)."""
        x, r = self.current_dev()
        self._x0, self._r0 = x, r
        self._y.zero_()
        self._My.zero_()
        self.best_norm = self._norm(self._r0)
        self.ncols = 0
        self.restart_count += 1


def _rm_step_dev(state: RmState, z_cand: torch.Tensor, D: DeviceBSR):
    """Device rm_step; returns (x, r) device tensors (solvers.py:559-625)."""
    ctx = state._ctx
    if state.ncols >= state.max_columns:
        state.restart()
    col = state.ncols
    z = state._Z[col]          # candidate lives in its would-be column
    w = state._W[col]
    z.copy_(z_cand)
    sc = state._sc
    D.spmv(z, w, norm_out=sc[0:1])                  # w = M z, ||w||^2
    if col > 0:
        Wv, Zv, coeff = state._W, state._Z, state._coeff
        for _ in range(2):   # two classical Gram-Schmidt passes
            ctx.gemv_t(Wv[:col], col, w, coeff)
            ctx.gemv_update2(Wv, Zv, col, coeff, w, z)
    ctx.dot(w, w, sc[1:2])
    s01 = _sync_read(sc[0:2])
    scale, norm_w = math.sqrt(s01[0]), math.sqrt(s01[1])
    if scale == 0.0 or norm_w <= DEPENDENT_CANDIDATE_RTOL * scale:
        state.last_dependent = True
        state.dependent_count += 1
        return state.current_dev()
    ctx.scale(norm_w, w, w, invert=True)
    ctx.scale(norm_w, z, z, invert=True)
    ctx.dot(w, state._r0, sc[2:3])                  # alpha = w . r0
    D.spmv(z, state._Mz)                            # exact image M z
    nat_check(ctx.lib.xdg_rm_update(
        state.n, state._r0.data_ptr(), state._My.data_ptr(),
        state._Mz.data_ptr(), sc[2:3].data_ptr(), state._My_new.data_ptr(),
        sc[3:4].data_ptr(), ctx.ws, ctx.stream), "rm_update")
    s23 = _sync_read(sc[2:4])
    alpha, rho = float(s23[0]), math.sqrt(s23[1])
    state.last_dependent = False
    if rho > state.best_norm:
        state.rejected_count += 1
        state.restart()
        return state.current_dev()
    state._alpha[col] = alpha
    ctx.axpy(1.0, z, state._y, a_dev=sc[2:3])       # y += alpha z
    state._My, state._My_new = state._My_new, state._My
    state.best_norm = rho
    state.ncols = col + 1
    return state.current_dev()


def nat_check(status, what):
    from . import _native as nat

    nat.check(status, what)


def rm_step(state: RmState, z_candidate, M) -> tuple:
    """Extend the search space by one candidate; returns (x, r, state) with
    the true residual of the new best point (solvers.py:559-625)."""
    if _length(z_candidate) != (state.n,):
        raise DimensionMismatchError("candidate length mismatch")
    ctx = state._ctx
    D = _device_operator(M, ctx)
    x, r = _rm_step_dev(state, _to_dev(z_candidate, ctx, copy=False), D)
    host = not _is_dev(z_candidate)
    return _out(x, not host), _out(r, not host), state


# ---------------------------------------------------------------------------
# multigrid over the aggregation hierarchy (solvers.py:632-749)


class _OmgContext:
    """Per-solve caches (solvers.py:632-666) plus their device twins."""

    def __init__(self, config: SolverConfig, entry_level: int = 1):
        self.config = config
        self.entry_level = entry_level
        self.partitions = {}
        self.transposes = {}
        self.coarse_factorization = {}
        self._dev = Context.get()

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


def _dev_norm(ctx: Context, v: torch.Tensor, slot: torch.Tensor) -> float:
    ctx.dot(v, v, slot)
    return math.sqrt(float(_sync_read(slot)[0]))


def _omg_dev(hierarchy, b: torch.Tensor, x0, config: SolverConfig, level: int,
             ctx_omg: _OmgContext):
    ctx = ctx_omg._dev
    lv = hierarchy.level(level)
    M = lv.matrix
    config.check_degree(lv.data.basis.degree)
    t_start = perf_counter()
    D = as_block_sparse(M).device(ctx)
    scal = torch.zeros(1, dtype=F64, device=ctx.device)
    n = M.shape[0]

    if level == hierarchy.num_levels or lv.restriction is None:
        x = ctx_omg.coarse_solver(hierarchy, level).apply_device(b)
        r = torch.empty_like(b)
        D.spmv(x, r, b=b, norm_out=scal)
        res = math.sqrt(float(_sync_read(scal)[0]))
        torch.cuda.synchronize(ctx.device)
        return x, SolverReport(solver="omg", iterations=0,
                               converged=res <= config.tolerance,
                               final_residual=res, residual_history=[res],
                               time_iterations=perf_counter() - t_start, dofs=n)

    x = torch.zeros_like(b) if x0 is None else _to_dev(x0, ctx)
    r = torch.empty_like(b)
    D.spmv(x, r, b=b)
    state = RmState(x, r, config.rm_max_columns)
    history = [state.best_norm]          # == ||r|| (same kernel, same data)
    partition = ctx_omg.partition(hierarchy, level)
    k_lo = config.k_lo_scalar
    R = as_block_sparse(lv.restriction)
    Rd = R.device(ctx)
    Rtd = ctx_omg.restriction_transpose(hierarchy, level).device(ctx)
    budget = (config.max_iterations if level == ctx_omg.entry_level
              else config.coarse_cycle_iterations)
    z = torch.empty_like(b)
    xf = torch.empty_like(b)
    rc = torch.empty(Rtd.nbr * Rtd.N, dtype=F64, device=ctx.device)
    it = 0
    while history[-1] > config.tolerance and it < budget:
        it += 1
        _schwarz_dev(M, D, r, partition, k_lo, ctx, z)
        x, r = _rm_step_dev(state, z, D)
        Rtd.spmv(r, rc)                                   # r_c = R^T r
        xc, _ = _omg_dev(hierarchy, rc, None, config, level + 1, ctx_omg)
        Rd.spmv(xc, xf)                                   # R x_c
        x, r = _rm_step_dev(state, xf, D)
        _schwarz_dev(M, D, r, partition, k_lo, ctx, z)
        x, r = _rm_step_dev(state, z, D)
        # ||r0 - My|| of the returned residual equals state.best_norm: every
        # exit of rm_step leaves r = r0 - My with best_norm its norm.
        history.append(state.best_norm)
    torch.cuda.synchronize(ctx.device)
    return x, SolverReport(solver="omg", iterations=it,
                           converged=history[-1] <= config.tolerance,
                           final_residual=history[-1], residual_history=history,
                           time_iterations=perf_counter() - t_start, dofs=n)


def ortho_mg_solve(hierarchy, b, x0=None, config: Optional[SolverConfig] = None,
                   level: int = 1, _context: Optional[_OmgContext] = None) -> tuple:
    """Orthonormalization multigrid (Alg. 4) on `level`; returns
    (solution, SolverReport); non-convergence is reported, not raised."""
    config = config or SolverConfig()
    ctx_omg = _context or _OmgContext(config, entry_level=level)
    lv = hierarchy.level(level)
    if _length(b) != (lv.matrix.shape[0],):
        raise DimensionMismatchError(
            f"rhs of length {_length(b)} against matrix {lv.matrix.shape}")
    bd = _to_dev(b, ctx_omg._dev)
    x, rep = _omg_dev(hierarchy, bd, x0, config, level, ctx_omg)
    return _out(x, _is_dev(b)), rep


# ---------------------------------------------------------------------------
# preconditioned GMRES (solvers.py:756-846)


def gmres_pmg_solve(M, b, config: Optional[SolverConfig] = None,
                    factorization_cache: Optional[dict] = None, *, dim: int,
                    x0=None) -> tuple:
    """Restarted GMRES, degree-separated preconditioner on the right, MGS
    orthogonalisation, Givens rotations; stops on the true residual."""
    from scipy.linalg import solve_triangular

    config = config or SolverConfig()
    cache = factorization_cache if factorization_cache is not None else {}
    if _length(b) != (M.shape[0],):
        raise DimensionMismatchError(f"rhs of length {_length(b)} against matrix {M.shape}")
    nb = M.row_layout.num_blocks
    all_cells = tuple(range(nb))
    k_lo = config.k_lo_scalar
    m = config.gmres_restart
    ctx = Context.get()
    t_start = perf_counter()
    D = _device_operator(M, ctx)
    modes_low = min(space_dimension(_normalize_k_lo(k_lo), dim), _uniform_block_size(M))
    plan = _pmg_plan(M, D, all_cells, modes_low, cache)
    bd = _to_dev(b, ctx)
    n = bd.numel()
    dev = ctx.device
    x = torch.zeros_like(bd) if x0 is None else _to_dev(x0, ctx)
    r = torch.empty_like(bd)
    sc = torch.zeros(m + 2, dtype=F64, device=dev)
    D.spmv(x, r, b=bd, norm_out=sc[0:1])
    beta = math.sqrt(float(_sync_read(sc[0:1])[0]))
    history = [beta]
    total = 0
    V = torch.empty(m + 1, n, dtype=F64, device=dev)
    Z = torch.empty(m, n, dtype=F64, device=dev)
    w = torch.empty(n, dtype=F64, device=dev)
    ycoef = torch.empty(m, dtype=F64, device=dev)

    while beta > config.tolerance and total < config.max_iterations:
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        ctx.scale(beta, r, V[0], invert=True)
        j = 0
        while j < m and total < config.max_iterations:
            total += 1
            plan.apply(V[j], Z[j])
            D.spmv(Z[j], w)
            for i in range(j + 1):                    # modified Gram-Schmidt
                ctx.dot(V[i], w, sc[i:i + 1])
                ctx.axpy(-1.0, V[i], w, a_dev=sc[i:i + 1])
            ctx.dot(w, w, sc[j + 1:j + 2])
            col = _sync_read(sc[: j + 2])
            H[: j + 1, j] = col[: j + 1]
            H[j + 1, j] = math.sqrt(col[j + 1])
            if H[j + 1, j] > 0.0:
                ctx.scale(H[j + 1, j], w, V[j + 1], invert=True)
            else:
                V[j + 1].zero_()
            for i in range(j):                        # stored rotations
                h_i = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = h_i
            denom = float(np.hypot(H[j, j], H[j + 1, j]))
            if denom == 0.0:
                raise SingularSystemError("preconditioned operator produced a zero column")
            cs[j] = H[j, j] / denom
            sn[j] = H[j + 1, j] / denom
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[j + 1, j] = 0.0
            estimate = abs(float(g[j + 1]))
            history.append(estimate)
            j += 1
            if estimate <= config.tolerance:
                break
        yv = solve_triangular(H[:j, :j], g[:j], check_finite=False)
        ycoef[:j].copy_(torch.from_numpy(-yv))
        # x = x + Z y   (as x -= Z (-y); negation is exact)
        ctx.gemv_update2(Z, None, j, ycoef, x, None)
        D.spmv(x, r, b=bd, norm_out=sc[0:1])
        beta = math.sqrt(float(_sync_read(sc[0:1])[0]))
        history[-1] = beta
    torch.cuda.synchronize(dev)
    rep = SolverReport(solver="gmres-pmg", iterations=total,
                       converged=beta <= config.tolerance, final_residual=beta,
                       residual_history=history,
                       time_iterations=perf_counter() - t_start, dofs=M.shape[0])
    return _out(x, _is_dev(b)), rep
