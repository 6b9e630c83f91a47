"""Pin the CPU oracle against the reference: golden fixtures written by
tests/golden/make_golden.py, which ran cutdg itself in the build container."""
import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_path
from oracle import cfg3, spmv

CASES = ["bench4", "cfg1", "sphere8p3"]


@pytest.mark.parametrize("case", CASES)
def test_oracle_spmv_bitexact_against_reference_matvec(case):
    z = np.load(golden_path(case))
    lam = 1
    while f"L{lam}_row_ptr" in z:
        p = f"L{lam}_"
        y = spmv.bsr_spmv(z[p + "row_ptr"], z[p + "col"], z[p + "val"], z[p + "x"])
        assert np.array_equal(y, z[p + "Mx"]), (case, lam)
        if p + "R_row_ptr" in z:
            yr = spmv.bsr_spmv(z[p + "R_row_ptr"], z[p + "R_col"], z[p + "R_val"],
                               z[p + "xc"])
            assert np.array_equal(yr, z[p + "Rxc"])
        lam += 1


def test_oracle_threads_do_not_change_bits():
    rp, col, val, x = cfg3.build(16)
    assert np.array_equal(spmv.bsr_spmv(rp, col, val, x, 1),
                          spmv.bsr_spmv(rp, col, val, x, 4))


def test_cfg3_recipe_counts_match_survey():
    rp, col, val, x = cfg3.build(16)
    y = spmv.bsr_spmv(rp, col, val, x)
    csr = sp.bsr_matrix((val, col, rp)).tocsr()
    assert np.array_equal(y, csr @ x)  # == scipy csr_matvec


def test_cfg3_package_pattern_equals_oracle_recipe():
    from paper_2003_02431_b200.synthetic import cfg3_pattern

    for n in (5, 12):
        rp, col, _, _ = cfg3.build(n)
        rows, cols, _, first, _ = cfg3_pattern(n)
        assert np.array_equal(cols, col)
        assert np.array_equal(np.bincount(rows, minlength=len(rp) - 1), np.diff(rp))


def test_cfg3_full_size_counts():
    from paper_2003_02431_b200.synthetic import cfg3_counts

    assert cfg3_counts(64) == (275251, 1853683)
