"""More reference runs for a chaotic iteration-count envelope (SURVEY.md
8(c) item 4): trials t0..t1-1 of make_golden.perturbed() for one case of
make_cfg5_golden / make_cfg4_golden, run with the REFERENCE solver on the
hierarchy its own assemble_case builds.  A K = 5 envelope of a count that
moves by hundreds of iterations under 1-ulp perturbations (cfg5 p=3 GMRES:
2927..3312) does not bound a sixth run of the reference itself; this script
widens K.  Writes tests/golden/<name>_env_<solver>_<t0>_<t1>.json; the
tests read every such file next to the fixture's own K = 5 list.

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \\
        python tests/golden/extend_envelope.py cfg5_10_p3 gmres 5 10
"""
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cutdg.bench import BenchCase, assemble_case, default_k_lo  # noqa: E402
from cutdg.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve  # noqa: E402
from make_golden import perturbed  # noqa: E402


def main(name, solver, t0, t1):
    assert name.startswith("cfg5_"), "cfg5 cases only"
    _, cells, pdeg = name.split("_")
    cells, p = int(cells), int(pdeg[1:])
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    case = BenchCase(dim=3, cells=cells, degree=p, levelset="sphere",
                     levelset_params={"center": tuple(c), "radius": 0.5},
                     mu_a=1.0, mu_b=1000.0, num_levels=3)
    k_lo = min(default_k_lo(p), p)
    cfg = (SolverConfig(tolerance=1e-8, max_iterations=3000, k_lo=k_lo, num_levels=3)
           if solver == "omg" else
           SolverConfig(tolerance=1e-8, max_iterations=4000, k_lo=k_lo, gmres_restart=50))
    asm = assemble_case(case)
    hier = asm.hierarchy
    lv = hier.level(1)
    b = np.asarray(lv.rhs, float)
    its = []
    for t in range(t0, t1):
        s = time.time()
        bt = perturbed(b, t)
        if solver == "omg":
            _, rep = ortho_mg_solve(hier, bt, None, cfg, 1)
        else:
            _, rep = gmres_pmg_solve(lv.matrix, bt, cfg, dim=3)
        its.append(int(rep.iterations))
        print(f"[{name}] {solver} trial {t}: {rep.iterations} ({time.time() - s:.0f}s)",
              flush=True)
    with open(os.path.join(HERE, f"{name}_env_{solver}_{t0}_{t1}.json"), "w") as f:
        json.dump({"case": name, "solver": solver, "trials": [t0, t1], "iterations": its}, f)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
