"""BASELINE config 4 at full size on ONE GPU: 3D 96^3, p=2, two seeded
spheres r=0.3 (union level set), mu 1:100, f = sin(pi x) sin(pi y) sin(pi z),
4-level hierarchy, built by this package's own setup (case.assemble_case;
the reference's setup at this size takes many hours -- SURVEY 8(d) cfg4),
then OMG (Schwarz smoother with PMG, 4 levels) and GMRES(50)-PMG to the
BASELINE 1e-10.  One JSON line per phase on stdout.

    CELLS=96 python tools/bench_cfg4.py [omg,gmres]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200 import solvers as S  # noqa: E402
from paper_2003_02431_b200.case import BenchCase, assemble_case  # noqa: E402
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.factor import warmup  # noqa: E402
from paper_2003_02431_b200.solvers import (  # noqa: E402
    SolverConfig, gmres_pmg_solve, ortho_mg_solve)

cells = int(os.environ.get("CELLS", "96"))
solvers = (sys.argv[1] if len(sys.argv) > 1 else "omg,gmres").split(",")
c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)  # make_cfg4_golden.py centres
case = BenchCase(dim=3, cells=cells, degree=2, levelset="spheres",
                 levelset_params={"centers": [tuple(-0.4 + c), tuple(0.4 - c)],
                                  "radius": 0.3}, mu_b=100.0, num_levels=4, source="sin",
                 workers=os.cpu_count() or 1)
t0 = time.perf_counter()
asm = assemble_case(case)
hier = asm.hierarchy
setup = time.perf_counter() - t0
lv = hier.level(1)
print(json.dumps({"case": f"cfg4 {cells}^3 p=2 (native setup)", "setup_s": round(setup, 2),
                  "phases": {k: round(v, 2) for k, v in asm.phase_times.items()},
                  "dofs_raw": int(len(asm.rhs)), "dofs_agglomerated": lv.num_dofs,
                  "level_blocks": [hier.level(i).data.num_blocks
                                   for i in range(1, hier.num_levels + 1)],
                  "nnzb_level1": int(lv.matrix.device().nnzb)}), flush=True)
warmup(Context.get())
torch.cuda.synchronize()
meta = {"omg": {"tolerance": 1e-10, "max_iterations": 3000, "k_lo": 1, "num_levels": 4},
        "gmres": {"tolerance": 1e-10, "max_iterations": 6000, "k_lo": 1, "gmres_restart": 50}}
for solver in solvers:
    cfg = SolverConfig(**meta[solver])
    torch.cuda.synchronize()
    try:
        if solver == "omg":
            octx = S._OmgContext(cfg, 1)
            x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1, octx)
            loop = dict(octx.last_loop)
            del octx
        else:
            x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=3)
            loop = dict(S.LAST_LOOP)
    except NotImplementedError as exc:  # e.g. the global low-order factor > HBM
        print(json.dumps({"case": f"cfg4 {cells}^3", "solver": solver,
                          "unsupported": str(exc)}), flush=True)
        continue
    finally:
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    t = rep.time_iterations
    print(json.dumps({"case": f"cfg4 {cells}^3", "solver": solver, "config": meta[solver],
                      "iterations": rep.iterations, "converged": rep.converged,
                      "final_residual": rep.final_residual, "solve_s": round(t, 3),
                      "dof_per_s": len(asm.rhs) / t, "ms_per_iteration": 1e3 * t / max(
                          rep.iterations, 1), "loop": loop}), flush=True)
