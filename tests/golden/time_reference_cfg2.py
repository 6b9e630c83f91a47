"""Time the REFERENCE solvers (cutdg) at full BASELINE config 2 in the build
container for a bounded number of iterations (CPU baseline for the bench's
cfg2 solve rows: per-iteration time and the lazy setup inside the solve
timer).  Writes tests/golden/reference_cfg2_timing.json.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/time_reference_cfg2.py
"""
import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from cutdg.bench import BenchCase, assemble_case  # noqa: E402
from cutdg.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    case = BenchCase(dim=3, cells=32, degree=3, levelset="sphere",
                     levelset_params={"center": tuple(c), "radius": 0.6},
                     mu_a=1.0, mu_b=1000.0, alpha=0.1, num_levels=3)
    t0 = time.time()
    asm = assemble_case(case)
    out = {"setup_s": time.time() - t0, "cores": os.cpu_count(),
           "threads": os.environ.get("OPENBLAS_NUM_THREADS")}
    H = asm.hierarchy
    lv = H.level(1)
    print(json.dumps(out), flush=True)
    for its in (1, 3):
        cfg = SolverConfig(tolerance=1e-10, max_iterations=its, k_lo=2, rm_max_columns=800,
                           num_levels=3)
        t0 = time.time()
        _, rep = ortho_mg_solve(H, lv.rhs, None, cfg, 1)
        out[f"omg_{its}it_s"] = time.time() - t0
        out[f"omg_{its}it_residual"] = rep.final_residual
        print(json.dumps(out), flush=True)
    for its in (1, 3):
        cfg = SolverConfig(tolerance=1e-10, max_iterations=its, k_lo=2, gmres_restart=50)
        t0 = time.time()
        _, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=3)
        out[f"gmres_{its}it_s"] = time.time() - t0
        print(json.dumps(out), flush=True)
    with open(os.path.join(HERE, "reference_cfg2_timing.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
