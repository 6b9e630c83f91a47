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


# ---- solver restatement (oracle/solvers_np.py) vs the reference ----------
import json  # noqa: E402

from oracle import solvers_np as so  # noqa: E402
from threadpoolctl import threadpool_limits  # noqa: E402


def _fixture(case):
    z = np.load(golden_path(case))
    return z, json.loads(bytes(z["meta"]).decode())


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3"])
def test_oracle_pmg_schwarz_rm_bitexact(case):
    z, meta = _fixture(case)
    h = so.hierarchy_from_npz(z, meta["dim"])
    for lam, lv in enumerate(h.levels, start=1):
        x = z[f"L{lam}_x"]
        nb = len(lv["rp"]) - 1
        for klo in range(3):
            key = f"L{lam}_pmg_klo{klo}"
            if key in z:
                F = so.PmgFactors(lv["rp"], lv["col"], lv["val"], np.arange(nb),
                                  so.modes_low(klo, meta["dim"], lv["N"]))
                assert np.array_equal(F.apply(x), z[key]), key
        for key in z.files:
            if key.startswith(f"L{lam}_T") and "_schwarz_klo" in key:
                tgt = int(key[len(f"L{lam}_T"):].split("_")[0])
                klo = int(key.rsplit("klo", 1)[1])
                ext, damp = so.schwarz_blocks(lv["adjacency"], lv["N"], max(tgt, lv["N"]))
                m = so.modes_low(klo, meta["dim"], lv["N"])
                facs = [so.PmgFactors(lv["rp"], lv["col"], lv["val"], e, m) for e in ext]
                assert np.array_equal(so.schwarz_apply(facs, damp, x), z[key]), key
    lv = h.levels[0]
    st = so.Rm(np.zeros(lv["M"].shape[0]), np.asarray(z["L1_rhs"]), 3)
    # the fixtures were generated with one BLAS thread (threaded dgemv
    # changes the summation order of W.T @ w)
    with threadpool_limits(1):
        for i, c in enumerate(z["rm_cands"]):
            xx, rr = st.step(c, lv["M"])
            assert np.array_equal(xx, z["rm_x"][i]) and np.array_equal(rr, z["rm_r"][i])


@pytest.mark.parametrize("case", ["bench4", "cfg1"])
@pytest.mark.parametrize("solver", ["gmres", "omg"])
def test_oracle_solves_reproduce_reference(case, solver):
    z, meta = _fixture(case)
    with threadpool_limits(1):
        x, it, _ = so.timed_solve(z, meta, solver)
    assert it == int(z[f"{solver}_iters"])
    assert np.array_equal(x, z[f"{solver}_x"])
