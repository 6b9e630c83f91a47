"""Distribution-level iteration parity: the GPU solver run on the SAME
+-1-ulp perturbations of b as the reference envelope (SURVEY 8(d) recipe)
must produce an iteration-count distribution that overlaps the
reference's: ranges intersect and medians agree within 10 %.  At tol 1e-10
(and for OMG at every tolerance) the reference itself is chaotic, so this is
the meaningful parity statement there; stable cases are covered exactly by
test_solvers_gpu.test_iterations_inside_reference_envelope."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_path

pytestmark = pytest.mark.gpu
K = 12


def perturbed(b, t):
    if t == 0:
        return b.copy()
    s = np.random.default_rng(100 + t).choice([-1.0, 1.0], size=len(b))
    return b * (1.0 + 2.2e-16 * s)


@pytest.mark.parametrize("solver,tol", [("omg", 1e-10), ("omg", 1e-8), ("gmres", 1e-10)])
def test_cfg1_iteration_distribution_matches_reference(solver, tol):
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve

    env_path = os.path.join(GOLDEN, "cfg1_env.npz")
    ref = np.load(env_path)[f"{solver}_tol{tol:.0e}"]
    z = np.load(golden_path("cfg1"))
    meta = json.loads(bytes(z["meta"]).decode())
    hier = load_hierarchy(z)
    lv = hier.level(1)
    cfgd = dict(meta[solver])
    cfgd["tolerance"] = tol
    cfg = SolverConfig(**cfgd)
    its = []
    for t in range(K):
        bt = perturbed(np.asarray(lv.rhs), t)
        if solver == "omg":
            _, rep = ortho_mg_solve(hier, bt, None, cfg, 1)
        else:
            _, rep = gmres_pmg_solve(lv.matrix, bt, cfg, dim=meta["dim"])
        assert rep.converged
        its.append(rep.iterations)
    its = np.array(its)
    assert its.min() <= ref.max() + 1 and its.max() >= ref.min() - 1, (sorted(its), sorted(ref))
    mg, mr = np.median(its), np.median(ref)
    assert abs(mg - mr) <= 0.10 * mr, (mg, mr, sorted(its), sorted(ref))
