"""Full-size reference hierarchies (tests/golden/large/*.npz, written by
tests/golden/make_large.py; git-ignored, ~0.1-1 GB): device SpMV / transfer
bit-exact and the Schwarz smoother <= 1e-10 vs the reference at 86k-690k
DOFs.  Skipped when the fixture is absent."""
import os

import numpy as np
import pytest
import torch

from conftest import GOLDEN

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def fixture(name):
    p = os.path.join(GOLDEN, "large", f"{name}.npz")
    if not os.path.exists(p):
        pytest.skip(f"{p} not generated")
    return np.load(p)


@pytest.mark.parametrize("name", ["s16p3", "cfg2"])
def test_large_spmv_transfer_schwarz(name):
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.schwarz import schwarz_partition
    from paper_2003_02431_b200.solvers import schwarz_apply

    z = fixture(name)
    hier = load_hierarchy(z)
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        D = lv.matrix.device()
        y = D.spmv(torch.from_numpy(z[f"L{lam}_x"]).cuda()).cpu().numpy()
        assert np.array_equal(y, z[f"L{lam}_Mx"]), lam
        if lv.restriction is not None:
            R = lv.restriction.device()
            assert np.array_equal(R.spmv(torch.from_numpy(z[f"L{lam}_xc"]).cuda()).cpu().numpy(),
                                  z[f"L{lam}_Rxc"])
    lv = hier.level(1)
    part = schwarz_partition(lv.graph, lv.data, max(2000, lv.data.block_size))
    assert np.array_equal(part.damping, z["L1_T2000_damping"])
    got = schwarz_apply(lv.matrix, z["L1_x"], part, 2)
    ref = z["L1_T2000_schwarz_klo2"]
    assert np.linalg.norm(got - ref) <= 1e-10 * np.linalg.norm(ref)
