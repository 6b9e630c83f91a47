"""Drop-in for the solver dispatch of cutdg.bench (bench.py:46, 209-236)
and its SpMV micro-benchmark (bench.py:326-352).

`solve_assembled(case, asm)` accepts the reference's own `BenchCase` and
assembled case (`asm.hierarchy`), or any object with the same attributes
(`case.solver`, `case.degree`, `case.dim`, `case.solver_config()`; a
hierarchy with `.level(1)`), and runs the selected solver on the B200.
"""
from __future__ import annotations

import statistics
from time import perf_counter

import numpy as np

from .blockmatrix import as_block_sparse
from .direct import direct_factor
from .errors import InvalidConfigError
from .solvers import SolverConfig, SolverReport, gmres_pmg_solve, ortho_mg_solve

SOLVER_IDS = ("direct", "omg", "gmres-pmg")
MATOPS_CSV_HEADER = "op,repetitions,median_ms,nonzero_rows"


def _config_of(case) -> SolverConfig:
    cfg = case.solver_config()
    if isinstance(cfg, SolverConfig):
        return cfg
    return SolverConfig(**{k: getattr(cfg, k) for k in (
        "tolerance", "max_iterations", "k_lo", "schwarz_target_dofs",
        "gmres_restart", "num_levels", "rm_max_columns",
        "coarse_cycle_iterations")})


def solve_assembled(case, asm):
    """Run the case's solver on the level-1 system; returns
    (solution on level 1, SolverReport with the setup phase times)."""
    if case.solver not in SOLVER_IDS:
        raise InvalidConfigError(f"unknown solver {case.solver!r}; choose from {SOLVER_IDS}")
    hier = asm.hierarchy
    lv = hier.level(1)
    config = _config_of(case)
    config.check_degree(case.degree)
    if case.solver == "direct":
        t0 = perf_counter()
        x = direct_factor(lv.matrix).apply(lv.rhs)
        dt = perf_counter() - t0
        M = as_block_sparse(lv.matrix)
        res = float(np.linalg.norm(lv.rhs - M.matvec(x)))
        report = SolverReport(solver="direct", iterations=0, converged=True,
                              final_residual=res, residual_history=[res],
                              time_iterations=dt, dofs=lv.num_dofs)
    elif case.solver == "omg":
        x, report = ortho_mg_solve(hier, lv.rhs, None, config, 1)
    else:
        x, report = gmres_pmg_solve(lv.matrix, lv.rhs, config, dim=case.dim)
    times = getattr(asm, "phase_times", {}) or {}
    report.time_basis_setup = times.get("basis", 0.0)
    report.time_matmat_setup = times.get("matmat", 0.0)
    return x, report


def micro_bench_matvec(M, repetitions: int = 20) -> list:
    """Median wall time of the device matvec on an assembled matrix
    (the matvec row of micro_bench_matops, bench.py:334-342)."""
    import torch

    if repetitions < 1:
        raise InvalidConfigError("repetitions must be >= 1")
    B = as_block_sparse(M)
    D = B.device()
    nonzero_rows = int(np.count_nonzero(np.diff(B.tocsr().indptr)))
    v = torch.ones(M.shape[1], dtype=torch.float64, device=D.ctx.device)
    y = D.spmv(v)
    times = []
    for _ in range(repetitions):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        D.spmv(v, y)
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return [["matvec", repetitions, f"{statistics.median(times):.6f}", nonzero_rows]]
