"""Benchmark cases and the setup pipeline (cutdg bench.py:67-206).

`assemble_case(case)` runs mesh -> cut-cell rules -> small-cell agglomeration
-> SIP assembly -> aggregation hierarchy, returning the solver-facing
`MultigridHierarchy` (hierarchy.py) whose level operators live in HBM.  It is
the reference's assemble_case (bench.py:165-206) with the bulk work moved:
cut-cell geometry on all host cores (worker processes), the raw operator
formed on the device from term lists (xdg_assemble_blocks), aggregate
carriers per cut aggregate on the host and once per shape for uncut ones,
Galerkin products on the device (xdg_galerkin).

Extensions beyond the reference's BenchCase, for BASELINE configs 4 and 5:
`levelset="spheres"` (union of balls, params centers/radius) and
`source="sin"` (f = sin(pi x) sin(pi y) sin(pi z)).
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .assembly import PieceIndex, PlainBasis, dirichlet_problem, sip_terms
from .blockmatrix import BlockSparseMatrix, uniform_layout
from .cutcells import classify_and_build
from .errors import InvalidConfigError
from .geometry import (
    CartesianMesh,
    LevelSet,
    UnionLevelSet,
    level_aggregates,
    small_cell_pairs,
)
from .hierarchy import HierarchyLevel, LevelInfo, MultigridHierarchy, _Basis
from .solvers import SolverConfig
from .transfer import (
    LevelBuilder,
    aggregate_graph,
    aggregation_level_data,
    assemble_device,
    build_restriction,
    galerkin_dev,
    initial_restriction,
    restrict_rhs,
)


SOLVER_IDS = ("direct", "omg", "gmres-pmg")  # bench.py:46


def default_alpha(degree: int) -> float:
    """bench.py:56-59."""
    return 0.1 if degree <= 3 else 0.3


def default_k_lo(degree: int) -> int:
    """bench.py:62-64."""
    return 1 if degree <= 3 else 3


@dataclass(frozen=True)
class BenchCase:
    """bench.py:67-136 (same fields and defaults) + `source`, `workers`."""

    dim: int = 3
    cells: int = 4
    degree: int = 2
    mu_a: float = 1.0
    mu_b: float = 1000.0
    alpha: Optional[float] = None
    levelset: str = "paper-benchmark"
    levelset_params: dict = field(default_factory=dict)
    solver: str = "omg"
    tolerance: float = 1e-10
    k_lo: Optional[int] = None
    num_levels: int = 2
    max_iterations: int = 1000
    schwarz_target_dofs: int = 2000
    gmres_restart: int = 30
    rm_max_columns: int = 200
    coarse_cycle_iterations: int = 2
    quad_depth: int = 3
    gauss_order: Optional[int] = None
    out: Optional[str] = None
    source: str = "one"
    workers: Optional[int] = None

    def __post_init__(self):
        if self.dim not in (2, 3):
            raise InvalidConfigError("dim must be 2 or 3")
        if self.cells < 1:
            raise InvalidConfigError("cells must be >= 1")
        if self.degree < 0:
            raise InvalidConfigError("degree must be >= 0")
        if self.solver not in SOLVER_IDS:
            raise InvalidConfigError(f"unknown solver {self.solver!r}; choose from {SOLVER_IDS}")
        if self.quad_depth < 0:
            raise InvalidConfigError("quad_depth must be >= 0")
        if self.source not in ("one", "sin"):
            raise InvalidConfigError(f"unknown source {self.source!r}")

    @property
    def resolved_alpha(self) -> float:
        return self.alpha if self.alpha is not None else default_alpha(self.degree)

    @property
    def resolved_k_lo(self) -> int:
        k_lo = self.k_lo if self.k_lo is not None else default_k_lo(self.degree)
        return min(k_lo, self.degree)

    @property
    def resolved_gauss_order(self) -> int:
        return self.gauss_order if self.gauss_order is not None else self.degree + 2

    def solver_config(self) -> SolverConfig:
        return SolverConfig(tolerance=self.tolerance, max_iterations=self.max_iterations,
                            k_lo=(self.resolved_k_lo,),
                            schwarz_target_dofs=self.schwarz_target_dofs,
                            gmres_restart=self.gmres_restart, num_levels=self.num_levels,
                            rm_max_columns=self.rm_max_columns,
                            coarse_cycle_iterations=self.coarse_cycle_iterations)


def make_level_set(name: str, params: Optional[dict] = None):
    """levelset.py:111-126 plus "spheres" (union of equal balls)."""
    params = dict(params or {})
    if name == "spheres":
        r = params.get("radius", 0.3)
        return UnionLevelSet([LevelSet("sphere", {"center": c, "radius": r})
                              for c in params["centers"]])
    if name not in ("sphere", "plane", "paper-benchmark", "benchmark"):
        raise InvalidConfigError(f"unknown level set name: {name!r}")
    return LevelSet(name, params)


def _sin_source(x):
    return np.sin(np.pi * x[:, 0]) * np.sin(np.pi * x[:, 1]) * (
        np.sin(np.pi * x[:, 2]) if x.shape[1] > 2 else 1.0)


@dataclass
class Assembled:
    cutmesh: object
    basis: PlainBasis
    pieces: PieceIndex
    matrix: BlockSparseMatrix      # raw system, device-resident
    rhs: np.ndarray
    hierarchy: MultigridHierarchy
    phase_times: dict
    terms: object = None


def build_hierarchy(cm, basis, pidx, raw_dev, rhs, level_groups, phase_times=None,
                    ctx=None) -> tuple:
    """build_hierarchy (transfer.py:456-522) over a device-resident raw
    operator.  `level_groups[l]` = aggregates of level l+1.  Returns
    (MultigridHierarchy, to_level1 BSR arrays)."""
    from .device import Context

    ctx = ctx or Context.get()
    times = phase_times if phase_times is not None else {}
    times.setdefault("basis", 0.0)
    times.setdefault("matmat", 0.0)
    N, mesh = basis.size, cm.mesh
    lb = LevelBuilder(cm, basis)
    t0 = time.perf_counter()
    lvl = aggregation_level_data(lb, level_groups[0])
    block_of = {(int(j), int(s)): b for b, (j, s) in enumerate(pidx.pieces)}
    R0 = initial_restriction(lvl, block_of, N)
    times["basis"] += time.perf_counter() - t0

    def galerkin(Md, pattern, R, nc):
        from .device import DeviceBSR

        Rd = DeviceBSR.from_arrays(R[0], R[1], R[2], N, nc, ctx)
        C, c_pat = galerkin_dev(Md, Rd, nc, ctx, pattern=pattern, r_pattern=(R[0], R[1]))
        return C, c_pat

    t0 = time.perf_counter()
    M, pat = galerkin(raw_dev, None, R0, lvl.num_blocks)
    b = restrict_rhs(R0, rhs, lvl.num_blocks, N)
    times["matmat"] += time.perf_counter() - t0
    datas, systems, transfers = [lvl], [(M, pat, b)], []
    for groups in level_groups[1:]:
        t0 = time.perf_counter()
        R, coarse = build_restriction(lb, datas[-1], groups)
        times["basis"] += time.perf_counter() - t0
        t0 = time.perf_counter()
        M, pat = galerkin(systems[-1][0], systems[-1][1], R, coarse.num_blocks)
        b = restrict_rhs(R, systems[-1][2], coarse.num_blocks, N)
        times["matmat"] += time.perf_counter() - t0
        transfers.append(R)
        datas.append(coarse)
        systems.append((M, pat, b))
    levels = []
    bas = _Basis(basis.degree, mesh.dim)
    for i, (d, (Md, _pat, bl)) in enumerate(zip(datas, systems)):
        lay = uniform_layout(d.num_blocks, N)
        Rm = None
        if i < len(transfers):
            nxt = datas[i + 1].num_blocks
            rp, col, val = transfers[i]
            Rm = BlockSparseMatrix.from_bsr(rp, col, val, lay, uniform_layout(nxt, N))
        levels.append(HierarchyLevel(
            data=LevelInfo(basis=bas, num_blocks=d.num_blocks),
            matrix=BlockSparseMatrix.from_device(Md, lay, lay), rhs=bl, restriction=Rm,
            graph=aggregate_graph(d, mesh)))
    meta = {"dim": mesh.dim, "num_levels": len(levels), "degree": basis.degree,
            "carrier_cache_hits": lb.cache_hits}
    return MultigridHierarchy(levels=levels, meta=meta), R0


def assemble_case(case: BenchCase, keep_terms: bool = False) -> Assembled:
    """bench.py:165-206 on the B200 pipeline (see module docstring).  Host
    BLAS runs single-threaded: the host work is many tiny dense products
    (multi-threaded BLAS costs ~100x on 20x20 solves); worker processes
    provide the parallelism."""
    try:
        from threadpoolctl import threadpool_limits
    except ImportError:  # pragma: no cover
        return _assemble_case(case, keep_terms)
    with threadpool_limits(1):
        return _assemble_case(case, keep_terms)


def _assemble_case(case: BenchCase, keep_terms: bool) -> Assembled:
    from .device import Context

    times: dict = {}
    t0 = time.perf_counter()
    ls = make_level_set(case.levelset, case.levelset_params)
    mesh = CartesianMesh([(-1.0, 1.0)] * case.dim, [case.cells] * case.dim)
    basis = PlainBasis(case.degree, case.dim)
    cm = classify_and_build(mesh, ls, case.quad_depth, case.resolved_gauss_order,
                            workers=case.workers)
    times["geometry"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    small = small_cell_pairs(cm.species_volume, mesh.cell_volume, mesh.adjacency(),
                             case.resolved_alpha)
    groups = level_aggregates(mesh, cm.species_volume, small, case.num_levels)
    times["agglomeration"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    src = _sin_source if case.source == "sin" else (lambda x: np.ones(len(x)))
    problem = dirichlet_problem(case.mu_a, case.mu_b, src, case.dim)
    terms = sip_terms(cm, basis, problem, groups[0])
    times["assembly_host"] = time.perf_counter() - t0
    ctx = Context.get()
    t0 = time.perf_counter()
    raw = assemble_device(terms, ctx)
    ctx_sync()
    times["assembly_device"] = time.perf_counter() - t0
    pidx = PieceIndex.build(cm.species_volume)
    H, R0 = build_hierarchy(cm, basis, pidx, raw, terms.rhs, groups, times, ctx)
    ctx_sync()
    lay = uniform_layout(pidx.num_blocks, basis.size)
    H.to_level1 = BlockSparseMatrix.from_bsr(
        R0[0], R0[1], R0[2], lay, uniform_layout(H.level(1).data.num_blocks, basis.size))
    return Assembled(cm, basis, pidx, BlockSparseMatrix.from_device(raw, lay, lay), terms.rhs,
                     H, times, terms if keep_terms else None)


def ctx_sync():
    import torch

    if torch.cuda.is_available():
        torch.cuda.synchronize()
