"""Reference iteration-count envelopes under +-1-ulp perturbations of b
(recipe 8(d)): trial 0 uses b, trial t >= 1 uses
b * (1 + 2.2e-16 s), s = default_rng(100 + t).choice([-1, 1], len(b)).
Runs the REFERENCE (cutdg) in the build container; writes
tests/golden/<case>_env.npz with, per (solver, tolerance), the list of
iteration counts.

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_envelope.py cfg1 [bench4 sphere8p3]
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cutdg.bench import assemble_case  # noqa: E402
from cutdg.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve  # noqa: E402
from make_golden import CASES, build_case, perturbed  # noqa: E402

PLAN = {
    "cfg1": {1e-10: 20, 1e-9: 20, 1e-8: 40},
    "bench4": {1e-10: 10, 1e-9: 5, 1e-8: 5},
    "sphere8p3": {1e-8: 10},
}


def main(name):
    spec = CASES[name]
    case = build_case(name)
    asm = assemble_case(case)
    hier = asm.hierarchy
    lv = hier.level(1)
    b = np.asarray(lv.rhs, float)
    out = {}
    for solver in ("gmres", "omg"):
        for tol, K in PLAN[name].items():
            cfgd = dict(spec[solver])
            cfgd["tolerance"] = tol
            cfg = SolverConfig(**cfgd)
            its = []
            t0 = time.time()
            for t in range(K):
                bt = perturbed(b, t)
                if solver == "omg":
                    _, rep = ortho_mg_solve(hier, bt, None, cfg, 1)
                else:
                    _, rep = gmres_pmg_solve(lv.matrix, bt, cfg, dim=case.dim)
                its.append(rep.iterations)
            out[f"{solver}_tol{tol:.0e}"] = np.array(its, np.int64)
            print(f"[{name}] {solver} tol={tol:.0e} K={K}: [{min(its)}, {max(its)}] "
                  f"{its} ({time.time() - t0:.0f}s)", flush=True)
    np.savez(os.path.join(HERE, f"{name}_env.npz"), **out)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        main(n)
