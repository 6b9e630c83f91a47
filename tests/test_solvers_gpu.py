"""Residual minimization, OMG and GMRES-PMG on the device vs the reference
(golden fixtures): parity protocol items 2-4."""
import json

import numpy as np
import pytest

from conftest import golden_path
from paper_2003_02431_b200.hierarchy import load_hierarchy
from paper_2003_02431_b200.solvers import (
    RmState,
    SolverConfig,
    gmres_pmg_solve,
    ortho_mg_solve,
    rm_step,
)

pytestmark = pytest.mark.gpu
SOL_TOL = 1e-8      # north_star: final solution within 1e-8 relative L2


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def load(case):
    z = np.load(golden_path(case))
    return z, json.loads(bytes(z["meta"]).decode()), load_hierarchy(z)


@pytest.mark.parametrize("case", ["bench4", "cfg1"])
def test_rm_step_sequence_matches_reference(case):
    z, meta, hier = load(case)
    lv = hier.level(1)
    b = lv.rhs
    state = RmState(np.zeros_like(b), b, 3)
    for i, cand in enumerate(z["rm_cands"]):
        x, r, state = rm_step(state, cand, lv.matrix)
        info = [state.ncols, int(state.last_dependent), state.dependent_count,
                state.rejected_count, state.restart_count]
        assert info == list(z["rm_info"][i]), (i, info, z["rm_info"][i])
        assert rel(x, z["rm_x"][i]) <= 1e-10, (i, rel(x, z["rm_x"][i]))
        assert rel(r, z["rm_r"][i]) <= 1e-10, (i, rel(r, z["rm_r"][i]))


@pytest.mark.parametrize("case", ["bench4", "cfg1"])
def test_omg_matches_reference(case):
    z, meta, hier = load(case)
    lv = hier.level(1)
    cfg = SolverConfig(**meta["omg"])
    x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1)
    assert rep.converged
    assert rel(x, z["omg_x"]) <= SOL_TOL
    assert rel(x, z["L1_direct_rhs"]) <= SOL_TOL
    h = rep.residual_history
    assert len(h) == rep.iterations + 1
    assert all(b <= a * (1 + 1e-12) for a, b in zip(h, h[1:]))
    assert rep.dofs == lv.num_dofs


@pytest.mark.parametrize("case", ["bench4", "cfg1"])
def test_gmres_matches_reference(case):
    z, meta, hier = load(case)
    lv = hier.level(1)
    cfg = SolverConfig(**meta["gmres"])
    x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=meta["dim"])
    assert rep.converged
    assert rel(x, z["gmres_x"]) <= SOL_TOL
    assert rel(x, z["L1_direct_rhs"]) <= SOL_TOL
    assert rep.residual_history[-1] == rep.final_residual


def test_omg_coarsest_is_direct_and_nonconvergence_reported():
    z, meta, hier = load("bench4")
    lv = hier.level(1)
    x, rep = ortho_mg_solve(hier, lv.rhs, None, SolverConfig(max_iterations=3, k_lo=1), 1)
    assert not rep.converged and rep.iterations == 3
    lc = hier.level(hier.num_levels)
    xc, repc = ortho_mg_solve(hier, lc.rhs, None, SolverConfig(), hier.num_levels)
    assert repc.iterations == 0 and repc.converged


def test_omg_respects_initial_guess():
    z, meta, hier = load("bench4")
    lv = hier.level(1)
    xd = z["L1_direct_rhs"]
    x, rep = ortho_mg_solve(hier, lv.rhs, xd.copy(),
                            SolverConfig(max_iterations=5, k_lo=1), 1)
    assert rep.converged and rep.iterations == 0 and np.allclose(x, xd)


def test_direct_factorization_matches_reference():
    from paper_2003_02431_b200.blockmatrix import direct_factor

    for case in ("bench4", "cfg1", "sphere8p3"):
        z, meta, hier = load(case)
        for lam in range(1, hier.num_levels + 1):
            lv = hier.level(lam)
            F = direct_factor(lv.matrix)
            x = F.apply(lv.rhs)
            assert rel(x, z[f"L{lam}_direct_rhs"]) <= 1e-9
            assert F.factor_count == 1


def test_dense_lu_inverse_apply_random_systems():
    """Triangular-inverse LU applies (one-CTA batched and whole-GPU) vs numpy."""
    import torch

    from paper_2003_02431_b200.device import Context
    from paper_2003_02431_b200.direct import DeviceDirect

    rng = np.random.default_rng(11)
    for n in (1, 37, 600, 2048, 5000):
        A = rng.standard_normal((n, n)) + n ** 0.5 * np.eye(n)
        b = rng.standard_normal(n)
        F = DeviceDirect(torch.from_numpy(A).cuda(), Context.get())
        x1 = F.apply(torch.from_numpy(b).cuda()).cpu().numpy()
        x2 = F.apply(torch.from_numpy(b).cuda()).cpu().numpy()
        assert np.array_equal(x1, x2)  # deterministic
        xr = np.linalg.solve(A, b)
        assert rel(x1, xr) <= 1e-12, (n, rel(x1, xr))


# ---- iteration counts vs the reference's own +-1-ulp envelopes ------------
# tests/golden/<case>_env.npz (make_envelope.py): K reference runs per
# (solver, tolerance) with b perturbed by +-1 ulp.  The bar is SURVEY 8(c)
# item 4 everywhere: [min - 1, max + 1] of the reference's own K = 10-40
# runs.  Where the reference is stable (envelope width <= 2: bench4
# everywhere, cfg1 GMRES at 1e-8/1e-9) that is the literal +-1 criterion;
# where the reference itself is chaotic (OMG at every tolerance, GMRES at
# 1e-10) K is large enough for the range to bound another run, and
# test_envelope_stats_gpu.py compares whole distributions.
import os  # noqa: E402

from conftest import GOLDEN  # noqa: E402


def _env_cases():
    out = []
    for case in ("bench4", "cfg1", "sphere8p3"):
        p = os.path.join(GOLDEN, f"{case}_env.npz")
        if os.path.exists(p):
            e = np.load(p)
            for k in e.files:
                solver, tol = k.split("_tol")
                out.append((case, solver, float(tol)))
    return out


@pytest.mark.parametrize("case,solver,tol", _env_cases())
def test_iterations_inside_reference_envelope(case, solver, tol):
    z, meta, hier = load(case)
    env = np.load(os.path.join(GOLDEN, f"{case}_env.npz"))[f"{solver}_tol{tol:.0e}"]
    lv = hier.level(1)
    cfgd = dict(meta[solver])
    cfgd["tolerance"] = tol
    cfg = SolverConfig(**cfgd)
    if solver == "omg":
        x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1)
    else:
        x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=meta["dim"])
    assert rep.converged
    # inside [min - 1, max + 1] of the reference's own
    # +-1-ulp envelope (K = 20-40 perturbed runs per tolerance)
    lo, hi = int(env.min()), int(env.max())
    assert lo - 1 <= rep.iterations <= hi + 1, (rep.iterations, sorted(env))
    assert rel(x, z["L1_direct_rhs"]) <= max(1e-8, 100 * tol)


def test_register_resident_mgs_is_bit_identical():
    """GMRES with the register-resident MGS kernel (mgs_reg_kernel, used
    from 32,768 unknowns: the 16^3 p=3 hierarchy) and with the streaming one
    (XDG_MGS_REG=0) gives identical histories and solutions (same arithmetic
    in the same order on the same grid)."""
    import subprocess
    import sys

    code = (
        "import hashlib, json, numpy as np\n"
        "from conftest import golden_path\n"
        "from paper_2003_02431_b200.hierarchy import load_hierarchy\n"
        "from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve\n"
        "z = np.load(golden_path('large/s16p3'))\n"
        "h = load_hierarchy(z)\n"
        "lv = h.level(1)\n"
        "x, r = gmres_pmg_solve(lv.matrix, np.asarray(lv.rhs), SolverConfig(tolerance=1e-8,"
        " max_iterations=300, k_lo=2, gmres_restart=50), dim=3)\n"
        "print(json.dumps([r.iterations, hashlib.sha1(np.asarray(x).tobytes()).hexdigest(),"
        " hashlib.sha1(np.asarray(r.residual_history).tobytes()).hexdigest()]))\n")
    here = os.path.dirname(os.path.abspath(__file__))
    if not os.path.exists(golden_path("large/s16p3")):
        pytest.skip("large/s16p3 fixture absent (tests/golden/make_large.py)")
    outs = []
    for flag in ("1", "0"):
        env = dict(os.environ, XDG_MGS_REG=flag,
                   PYTHONPATH=os.pathsep.join([here, os.path.dirname(here)]))
        p = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                           text=True, timeout=600, cwd=here)
        assert p.returncode == 0, p.stderr[-2000:]
        outs.append(json.loads(p.stdout.strip().splitlines()[-1]))
    assert outs[0] == outs[1]
