"""Setup row SURVEY 8(f)#2 on the device: the raw operator formed by
xdg_assemble_blocks (bit-identical to the host evaluation of the same term
lists), the whole assemble_case pipeline (device assembly + device Galerkin
products) against the reference's level operators, and solves on the natively
assembled hierarchy against the reference's solutions and iteration
envelopes."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_path
from paper_2003_02431_b200.case import assemble_case
from paper_2003_02431_b200.hierarchy import fixture_array
from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve
from paper_2003_02431_b200.transfer import assemble_device
from test_setup import case_of, host_setup

pytestmark = pytest.mark.gpu
# max |dM| / max |M| vs the reference's fixtures; sphere8p3 (p=3): the
# reference reproduces its own fixture only to 2.5e-10.
TOL = {"bench4": 1e-12, "cfg1": 1e-12, "sphere8p3": 1e-9}
_ASM = {}


def native(name):
    if name not in _ASM:
        c, z = case_of(name)
        _ASM[name] = (c, z, assemble_case(c))
    return _ASM[name]


@pytest.mark.parametrize("name", ["bench4", "cfg1"])
def test_assemble_kernel_bit_exact(name):
    *_, T = host_setup(name)
    rp, col, val = assemble_device(T).to_host_rowmajor()
    assert np.array_equal(rp, T.row_ptr) and np.array_equal(col, T.col)
    assert np.array_equal(val, T.evaluate_host())


@pytest.mark.parametrize("name", ["bench4", "cfg1", "sphere8p3"])
def test_assemble_case_levels(name):
    c, z, A = native(name)
    H = A.hierarchy
    assert H.num_levels == c.num_levels
    for lam in range(1, c.num_levels + 1):
        p = f"L{lam}_"
        lv = H.level(lam)
        rp, col, val = lv.matrix.bsr_arrays()
        assert np.array_equal(rp, z[p + "row_ptr"]) and np.array_equal(col, z[p + "col"])
        ref = fixture_array(z, p + "val")
        err = np.abs(val - ref).max() / np.abs(ref).max()
        assert err <= TOL[name], (lam, err)
        rr = z[p + "rhs"]
        assert np.abs(lv.rhs - rr).max() <= 1e3 * TOL[name] * np.abs(rr).max()
        adj = np.array([v for a in lv.graph.adjacency for v in a], np.int64)
        assert np.array_equal(adj, z[p + "adj"])
        ptr, flat = lv.graph.csr  # the array copy schwarz_partition reads
        srt = np.array([v for a in lv.graph.adjacency for v in sorted(a)], np.int64)
        assert np.array_equal(flat, srt)
        assert np.array_equal(np.diff(ptr), [len(a) for a in lv.graph.adjacency])


def _slack(env):
    lo, hi = int(env.min()), int(env.max())
    return 1 if hi - lo <= 2 else max(1, int(round(0.10 * np.median(env))))


@pytest.mark.parametrize("name,solver", [("bench4", "omg"), ("bench4", "gmres"),
                                         ("cfg1", "omg"), ("cfg1", "gmres")])
def test_solve_on_native_hierarchy(name, solver):
    c, z, A = native(name)
    meta = json.loads(bytes(z["meta"]).decode())
    H = A.hierarchy
    lv = H.level(1)
    cfg = SolverConfig(**meta[solver])
    if solver == "omg":
        x, rep = ortho_mg_solve(H, lv.rhs, None, cfg, 1)
    else:
        x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=c.dim)
    assert rep.converged
    ref = z["L1_direct_rhs"]
    assert np.linalg.norm(x - ref) <= 1e-8 * np.linalg.norm(ref)
    p = os.path.join(GOLDEN, f"{name}_env.npz")
    key = f"{solver}_tol{cfg.tolerance:.0e}"
    if os.path.exists(p) and key in np.load(p).files:
        env = np.load(p)[key]
        s = _slack(env)
        assert int(env.min()) - s <= rep.iterations <= int(env.max()) + s, (rep.iterations, sorted(env))
    else:
        ref_it = int(z[f"{solver}_iters"])
        assert abs(rep.iterations - ref_it) <= max(1, int(0.1 * ref_it)), (rep.iterations, ref_it)
