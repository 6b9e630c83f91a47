"""Drop-in for cutdg.bench: the solver dispatch (bench.py:46, 209-236), case
runs and sweeps with their CSV rows (bench.py:239-323), the matrix-operation
micro-benchmark (bench.py:326-359) and the MatrixMarket export (362-368),
over this package's setup pipeline (case.py) and B200 solvers.

`solve_assembled(case, asm)` accepts the reference's own `BenchCase` and
assembled case (`asm.hierarchy`), or any object with the same attributes
(`case.solver`, `case.degree`, `case.dim`, `case.solver_config()`; a
hierarchy with `.level(1)`), and runs the selected solver on the B200.
"""
from __future__ import annotations

import csv
import io
import statistics
from dataclasses import dataclass, replace
from time import perf_counter
from typing import Optional

import numpy as np

from .blockmatrix import as_block_sparse
from .direct import direct_factor
from .errors import CutDgError, InvalidConfigError
from .solvers import SolverConfig, SolverReport, gmres_pmg_solve, ortho_mg_solve

SOLVER_IDS = ("direct", "omg", "gmres-pmg")
SWEEP_CSV_HEADER = ("grid,k,dofs,solver,iterations,converged,setup_basis_ms,"
                    "setup_matmat_ms,solve_ms,final_residual,l2_error")
MATOPS_CSV_HEADER = "op,repetitions,median_ms,nonzero_rows"

from .case import BenchCase, assemble_case  # noqa: E402  (bench.py:68-206)


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


# ---------------------------------------------------------------------------
# case runs, sweeps, micro-benchmark, export (bench.py:140-380)

@dataclass
class CaseResult:
    """bench.py:140-151."""

    report: SolverReport
    dofs_raw: int
    dofs_agglomerated: int
    l2_error: Optional[float] = None

    @property
    def converged(self) -> bool:
        return self.report.converged


def run_case(case, exact=None) -> CaseResult:
    """Build and solve one case (bench.py:239-259).  The broken-L2 error
    against an exact solution (`exact`) needs the reference's cut-cell
    quadrature evaluator, which is outside this package's scope."""
    if exact is not None:
        raise NotImplementedError("l2 error evaluation is not part of the B200 solver path")
    asm = assemble_case(case)
    _x, report = solve_assembled(case, asm)
    return CaseResult(report=report, dofs_raw=int(len(asm.rhs)),
                      dofs_agglomerated=asm.hierarchy.level(1).num_dofs)


def _sweep_row(case, result: Optional[CaseResult], error: str = "") -> list:
    """One SWEEP_CSV_HEADER row (bench.py:262-282): same fields, formats."""
    grid = f"{case.cells}^{case.dim}"
    if result is None:
        return [grid, case.degree, "", case.solver, 0, False, "", "", "", "", error]
    rep = result.report
    return [grid, case.degree, result.dofs_raw, case.solver, rep.iterations, rep.converged,
            f"{rep.time_basis_setup * 1e3:.3f}", f"{rep.time_matmat_setup * 1e3:.3f}",
            f"{rep.time_iterations * 1e3:.3f}", f"{rep.final_residual:.6e}",
            "" if result.l2_error is None else f"{result.l2_error:.6e}"]


def run_sweep(grids, degrees, solvers, base_case=None, out: Optional[str] = None) -> list:
    """Rows per (grid, degree, solver), one assembly per (grid, degree); a
    failing case is recorded in its row and the sweep continues
    (bench.py:285-323)."""
    if not grids or not degrees or not solvers:
        raise InvalidConfigError("sweep needs grids, degrees, and solvers")
    base = base_case or BenchCase()
    rows = []
    for n in grids:
        for k in degrees:
            asm = None
            for solver in solvers:
                case = replace(base, cells=int(n), degree=int(k), solver=solver)
                try:
                    if asm is None:
                        asm = assemble_case(case)
                    _x, report = solve_assembled(case, asm)
                    rows.append(_sweep_row(case, CaseResult(
                        report=report, dofs_raw=int(len(asm.rhs)),
                        dofs_agglomerated=asm.hierarchy.level(1).num_dofs)))
                except CutDgError as exc:
                    rows.append(_sweep_row(case, None, error=str(exc)))
    if out:
        with open(out, "w", newline="") as fh:
            w = csv.writer(fh)
            w.writerow(SWEEP_CSV_HEADER.split(","))
            w.writerows(rows)
    return rows


def micro_bench_matops(case, repetitions: int = 20) -> list:
    """Device matvec (median over `repetitions`, CUDA events) and the
    aggregation triple product R0^T M R0 (wall time through the public
    galerkin_restrict) on the case's raw system (bench.py:326-352)."""
    from .transfer import galerkin_restrict

    if repetitions < 1:
        raise InvalidConfigError("repetitions must be >= 1")
    asm = assemble_case(case)
    rows = micro_bench_matvec(asm.matrix, repetitions)
    t0 = perf_counter()
    galerkin_restrict(asm.matrix, None, asm.hierarchy.to_level1)
    rows.append(["matmat", 1, f"{(perf_counter() - t0) * 1e3:.6f}", rows[0][3]])
    return rows


def write_matops_csv(rows: list, out: str) -> None:
    """bench.py:355-359."""
    with open(out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(MATOPS_CSV_HEADER.split(","))
        w.writerows(rows)


def export_case_matrix(case, path: str) -> int:
    """Assemble and write the level-1 matrix as MatrixMarket coordinate
    (bench.py:362-368); returns its dimension."""
    from .blockmatrix import write_matrix_market

    asm = assemble_case(case)
    lv = asm.hierarchy.level(1)
    write_matrix_market(path, lv.matrix)
    return lv.num_dofs


def format_rows(header: str, rows: list) -> str:
    """bench.py:371-376."""
    buf = io.StringIO()
    w = csv.writer(buf)
    w.writerow(header.split(","))
    w.writerows(rows)
    return buf.getvalue()
