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


@pytest.mark.parametrize("name", ["s16p3", "cfg2"])
def test_gmres_pmg_full_size_true_residual_and_omg_agreement(name):
    """Full-size GMRES(50)-PMG (k_lo = 2; the cfg2 global low-order system
    is the 336,610-unknown multifrontal factor): converged, its true
    residual recomputed with the oracle SpMV (bit-identical to the
    reference matvec) at the tolerance's roundoff floor, and the solution
    equal to the converged OMG solution to 1e-8 (both solve the same
    system to an absolute residual of 1e-10)."""
    from oracle import spmv
    from paper_2003_02431_b200.hierarchy import fixture_array, load_hierarchy
    from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve

    z = fixture(name)
    meta = json.loads(bytes(z["meta"]).decode())
    hier = load_hierarchy(z)
    lv = hier.level(1)
    b = np.asarray(lv.rhs)
    gcfg = dict(meta["gmres"], max_iterations=20000)
    xg, rg = gmres_pmg_solve(lv.matrix, b, SolverConfig(**gcfg), dim=meta["dim"])
    assert rg.converged and rg.final_residual <= gcfg["tolerance"]
    assert rg.residual_history[-1] == rg.final_residual
    r = b - spmv.bsr_spmv(z["L1_row_ptr"], z["L1_col"], fixture_array(z, "L1_val"), xg,
                          spmv.max_threads())
    assert np.linalg.norm(r) <= 1e-8 * np.linalg.norm(b)
    xo, ro = ortho_mg_solve(hier, b, None, SolverConfig(**meta["omg"]), 1)
    assert ro.converged
    d = np.linalg.norm(xg - xo) / np.linalg.norm(xo)
    print(f"{name}: gmres {rg.iterations} it, omg {ro.iterations} it, |xg - xo|/|xo| = {d:.3e}")
    assert d <= 1e-8


def test_cfg2_low_order_multifrontal_backward_error():
    """The cfg2 GMRES-PMG global low-order system (33,661 blocks x 10 modes
    = 336,610 unknowns, k_lo = 2) factored by the device multifrontal LU:
    b = A x_true with the oracle SpMV, x = xdg_mf_solve(b); normwise
    backward error <= 5e-14 (measured: 1.0e-14 = 46 eps at n = 336,610; a
    partial-pivoting LU's bound is O(n eps)) and forward error bounded like a
    partial-pivoting LU's (eps cond(A))."""
    import torch

    from oracle import spmv
    from paper_2003_02431_b200.device import Context, DeviceBSR
    from paper_2003_02431_b200.direct import SparseDirect
    from paper_2003_02431_b200.hierarchy import fixture_array

    z = fixture("cfg2")
    rp, col = z["L1_row_ptr"], z["L1_col"]
    m = 10  # modes_low(k_lo=2, dim=3)
    val = np.ascontiguousarray(fixture_array(z, "L1_val")[:, :m, :m])
    nb = len(rp) - 1
    assert nb * m == 336_610
    ctx = Context.get()
    D = DeviceBSR.from_arrays(rp, col, val, m, nb, ctx)
    sd = SparseDirect(D, ctx)
    rng = np.random.default_rng(7)
    x_true = rng.standard_normal(nb * m)
    b = spmv.bsr_spmv(rp, col, val, x_true, spmv.max_threads())
    got = sd.apply(torch.from_numpy(b).to(ctx.device)).cpu().numpy()
    r = b - spmv.bsr_spmv(rp, col, val, got, spmv.max_threads())
    a_inf = np.abs(val).sum(axis=2)  # row sums of |A| per block row
    rows = np.repeat(np.arange(nb), np.diff(rp))
    rowsum = np.zeros((nb, m))
    np.add.at(rowsum, rows, a_inf)
    norm_a = rowsum.max()
    berr = np.abs(r).max() / (norm_a * np.abs(got).max() + np.abs(b).max())
    ferr = np.linalg.norm(got - x_true) / np.linalg.norm(x_true)
    print(f"cfg2 low-order: n = {nb * m}, factor {sd.mf.factor_bytes / 1e9:.2f} GB, "
          f"backward {berr:.3e}, forward {ferr:.3e}")
    assert berr <= 5e-14, berr
    assert ferr <= 1e-6, ferr
