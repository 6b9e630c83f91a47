"""Galerkin coarse operator R^T M R on the device vs the
reference: every coarse level matrix of the golden hierarchies IS the
reference's galerkin_restrict(M_fine, R) (transfer.py:496-500), and the
Table-2 instance (make_matops.py) stores the reference's R0^T M R0.
Reference test tolerance: 1e-11 vs a dense triple product
(test_transfer.py:166-190)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_path
from paper_2003_02431_b200.hierarchy import fixture_array, load_hierarchy

pytestmark = pytest.mark.gpu
TOL = 1e-11


def _compare(Mc, rp, col, val):
    r, c, v = Mc.bsr_arrays()
    assert np.array_equal(r, rp) and np.array_equal(c, col)
    scale = np.abs(val).max()
    assert np.abs(v - val).max() <= TOL * scale, np.abs(v - val).max() / scale


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3", "large/s16p3"])
def test_galerkin_levels_match_reference(case):
    from paper_2003_02431_b200.transfer import galerkin_restrict

    p = golden_path(case)
    if not os.path.exists(p):
        pytest.skip(f"{p} absent")
    z = np.load(p)
    hier = load_hierarchy(z)
    for lam in range(1, hier.num_levels):
        lv = hier.level(lam)
        Mc, bc = galerkin_restrict(lv.matrix, lv.rhs, lv.restriction)
        q = f"L{lam + 1}_"
        _compare(Mc, z[q + "row_ptr"], z[q + "col"], fixture_array(z, q + "val"))
        ref_b = z[q + "rhs"]
        assert np.abs(bc - ref_b).max() <= TOL * np.abs(ref_b).max()


@pytest.mark.parametrize("name", ["matops_4_k3", "matops_6_k5"])
def test_galerkin_table2_instance(name):
    from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout
    from paper_2003_02431_b200.transfer import galerkin_restrict

    p = os.path.join(GOLDEN, "large", f"{name}.npz")
    if not os.path.exists(p):
        pytest.skip(f"{p} absent")
    z = np.load(p)

    def mat(prefix, ncols):
        rp = z[prefix + "_row_ptr"]
        val = fixture_array(z, prefix + "_val")
        N = val.shape[1]
        return BlockSparseMatrix.from_bsr(rp, z[prefix + "_col"], val,
                                          uniform_layout(len(rp) - 1, N),
                                          uniform_layout(ncols, N))

    M = mat("M", int(z["M_ncols"]))
    R0 = mat("R0", int(z["R0_ncols"]))
    Mc, _ = galerkin_restrict(M, None, R0)
    _compare(Mc, z["Mc_row_ptr"], z["Mc_col"], fixture_array(z, "Mc_val"))
