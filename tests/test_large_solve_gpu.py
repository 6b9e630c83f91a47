"""Full-size solve parity (BASELINE config 2, 32^3 p=3, 690k DOFs; and the
16^3 p=3 hierarchy).  A full reference solve there takes hours on a CPU, so:
  * the first OMG iterations are compared with the CPU oracle
    (oracle/solvers_np.py, bit-identical to the reference on every pinned
    case, tests/test_oracle.py): residual histories and iterates agree to
    roundoff before the solver's chaotic branches can diverge;
  * the converged GPU solution's true residual ||b - M x|| is recomputed on
    the host with the oracle SpMV (bit-identical to the reference matvec)
    and must meet the tolerance.
Skipped when the serialized hierarchy (tests/golden/large) is absent."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def fixture(name):
    p = os.path.join(GOLDEN, "large", f"{name}.npz")
    if not os.path.exists(p):
        pytest.skip(f"{p} absent")
    return np.load(p)


@pytest.mark.parametrize("name", ["s16p3", "cfg2"])
def test_first_omg_iterations_match_oracle(name):
    from threadpoolctl import threadpool_limits

    from oracle import solvers_np as so
    from paper_2003_02431_b200.hierarchy import fixture_array, load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve

    z = fixture(name)
    meta = json.loads(bytes(z["meta"]).decode())
    K = 3
    cfgd = dict(meta["omg"])
    cfgd["max_iterations"] = K
    hier = load_hierarchy(z)
    x_gpu, rep = ortho_mg_solve(hier, hier.level(1).rhs, None, SolverConfig(**cfgd), 1)

    class Z(dict):  # oracle reader over the deduplicated fixture
        files = property(lambda self: list(self.keys()))

    zz = Z()
    for k in z.files:
        if k.endswith("__uniq"):
            base = k[: -len("__uniq")]
            zz[base] = fixture_array(z, base)
        elif not k.endswith("__idx"):
            zz[k] = z[k]
    h = so.hierarchy_from_npz(zz, meta["dim"])
    ocfg = dict(tolerance=1e-10, schwarz_target_dofs=2000, rm_max_columns=200,
                coarse_cycle_iterations=2)
    ocfg.update(meta["omg"])
    ocfg["max_iterations"] = K
    ocfg["k_lo"] = int(ocfg["k_lo"])
    with threadpool_limits(1):
        x_cpu, it, hist = so.omg(h, np.asarray(zz["L1_rhs"], float), ocfg)
    assert rep.iterations == it == K
    hist_gpu = np.array(rep.residual_history)
    hist_rel = np.abs(hist_gpu - np.array(hist)) / np.array(hist)
    x_rel = np.linalg.norm(x_gpu - x_cpu) / np.linalg.norm(x_cpu)
    print(f"{name}: history rel diff {hist_rel.max():.3e}, iterate rel diff {x_rel:.3e}")
    # dense LU vs SuperLU low-order solves differ by up to ~1e-12 per PMG
    # application at cond ~1e7; three RM-accelerated
    # cycles keep the iterates within 1e-8
    assert hist_rel.max() <= 1e-8, (hist_gpu, hist)
    assert x_rel <= 1e-8


@pytest.mark.parametrize("name", ["s16p3", "cfg2"])
def test_converged_solution_true_residual(name):
    from oracle import spmv
    from paper_2003_02431_b200.hierarchy import fixture_array, load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve

    z = fixture(name)
    meta = json.loads(bytes(z["meta"]).decode())
    hier = load_hierarchy(z)
    b = np.asarray(hier.level(1).rhs)
    cfg = SolverConfig(**meta["omg"])
    x, rep = ortho_mg_solve(hier, b, None, cfg, 1)
    assert rep.converged
    r = b - spmv.bsr_spmv(z["L1_row_ptr"], z["L1_col"], fixture_array(z, "L1_val"), x,
                          spmv.max_threads())
    res = np.linalg.norm(r)
    # The solver (like the reference, solvers.py:493-501, 546) reports the
    # tracked residual r0 - M y of exact images, which reaches tol 1e-10;
    # the recomputed b - M x sits at the roundoff floor eps ||M|| ||x||
    # (~2e-9 at these sizes), so it is checked relative to b.
    print(f"{name}: tracked {rep.final_residual:.3e}  true {res:.3e}")
    assert rep.final_residual <= cfg.tolerance
    assert res <= 1e-8 * np.linalg.norm(b), res
