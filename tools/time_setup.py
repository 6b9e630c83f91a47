"""Time the native setup pipeline (case.assemble_case) and optionally a solve
on the hierarchy it builds.

    python tools/time_setup.py --cells 32 --degree 3 [--levels 3] [--solve omg]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=32)
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--levels", type=int, default=3)
    ap.add_argument("--dim", type=int, default=3)
    ap.add_argument("--levelset", default="sphere")
    ap.add_argument("--radius", type=float, default=0.6)
    ap.add_argument("--mu-b", type=float, default=1000.0)
    ap.add_argument("--source", default="one")
    ap.add_argument("--solve", default="")
    ap.add_argument("--tol", type=float, default=1e-10)
    ap.add_argument("--k-lo", type=int, default=None)
    ap.add_argument("--max-it", type=int, default=3000)
    ap.add_argument("--rm-cols", type=int, default=200)
    ap.add_argument("--restart", type=int, default=50)
    a = ap.parse_args()
    from paper_2003_02431_b200.case import BenchCase, assemble_case
    from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve

    c = np.random.default_rng(0).uniform(-0.1, 0.1, a.dim)
    if a.levelset == "spheres":
        params = {"centers": [tuple(-0.4 + c), tuple(0.4 - c)], "radius": a.radius}
    else:
        params = {"center": tuple(c), "radius": a.radius}
    case = BenchCase(dim=a.dim, cells=a.cells, degree=a.degree, levelset=a.levelset,
                     levelset_params=params, mu_b=a.mu_b, num_levels=a.levels,
                     source=a.source)
    t0 = time.perf_counter()
    A = assemble_case(case)
    setup = time.perf_counter() - t0
    H = A.hierarchy
    out = {"cells": a.cells, "degree": a.degree, "levels": a.levels, "setup_s": round(setup, 3),
           "phases": {k: round(v, 3) for k, v in A.phase_times.items()},
           "raw_dofs": int(len(A.rhs)), "L1_dofs": H.level(1).num_dofs,
           "level_blocks": [H.level(l).data.num_blocks for l in range(1, H.num_levels + 1)],
           "cut_cells": len(A.cutmesh.interface_rules), "cache_hits": H.meta["carrier_cache_hits"]}
    for solver in [v for v in a.solve.split(",") if v]:
        lv = H.level(1)
        cfg = SolverConfig(tolerance=a.tol, max_iterations=a.max_it,
                           k_lo=(case.resolved_k_lo if a.k_lo is None else a.k_lo,),
                           num_levels=a.levels, rm_max_columns=a.rm_cols,
                           gmres_restart=a.restart)
        from paper_2003_02431_b200 import solvers as S

        t0 = time.perf_counter()
        if solver == "omg":
            octx = S._OmgContext(cfg, 1)
            x, rep = ortho_mg_solve(H, lv.rhs, None, cfg, 1, octx)
            loop = dict(octx.last_loop)
        else:
            x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=a.dim)
            loop = dict(S.LAST_LOOP)
        dt = time.perf_counter() - t0
        out[solver] = dict(solve_s=round(dt, 3), iterations=rep.iterations,
                           converged=rep.converged, final_residual=rep.final_residual,
                           dof_per_s=out["raw_dofs"] / rep.time_iterations,
                           loop_s=loop.get("seconds"),
                           loop_GBs=loop.get("bytes", 0) / max(loop.get("seconds", 1), 1e-12)
                           / 1e9)
        print(json.dumps(out), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
