"""Degree-separated preconditioner and Schwarz smoother on the device vs the
reference (golden fixtures) -- parity protocol item 2: <= 1e-10 relative
(two exact LU implementations differ by up to ~1.7e-12)."""
import json
import warnings

import numpy as np
import pytest
import torch

from conftest import golden_path
from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout
from paper_2003_02431_b200.errors import (
    DimensionMismatchError,
    InvalidConfigError,
    SingularSystemError,
)
from paper_2003_02431_b200.hierarchy import load_hierarchy
from paper_2003_02431_b200.schwarz import schwarz_partition
from paper_2003_02431_b200.solvers import pmg_apply, schwarz_apply

pytestmark = pytest.mark.gpu
TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3"])
def test_pmg_and_schwarz_match_reference(case):
    z = np.load(golden_path(case))
    meta = json.loads(bytes(z["meta"]).decode())
    hier = load_hierarchy(z)
    checked = 0
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        x = z[f"L{lam}_x"]
        nb = lv.matrix.row_layout.num_blocks
        for klo in range(3):
            key = f"L{lam}_pmg_klo{klo}"
            if key in z:
                got = pmg_apply(lv.matrix, x, klo, range(nb), {}, dim=meta["dim"])
                assert rel(got, z[key]) <= TOL, (key, rel(got, z[key]))
                checked += 1
        for key in z.files:
            if key.startswith(f"L{lam}_T") and "_schwarz_klo" in key:
                tgt = int(key[len(f"L{lam}_T"):].split("_")[0])
                klo = int(key.rsplit("klo", 1)[1])
                part = schwarz_partition(lv.graph, lv.data, max(tgt, lv.data.block_size))
                got = schwarz_apply(lv.matrix, x, part, klo)
                assert rel(got, z[key]) <= TOL, (key, rel(got, z[key]))
                checked += 1
    assert checked >= 3


# ---- reference unit-test semantics (test_solvers.py:194-299) -------------

def random_block_spd(num_blocks, size, seed=20240817, block_diagonal=False):
    rng = np.random.default_rng(seed)
    n = num_blocks * size
    if block_diagonal:
        A = np.zeros((n, n))
        for c in range(num_blocks):
            Q = rng.normal(size=(size, size))
            sl = slice(c * size, (c + 1) * size)
            A[sl, sl] = Q @ Q.T + size * np.eye(size)
    else:
        Q = rng.normal(size=(n, n))
        A = Q @ Q.T + n * np.eye(n)
    M = BlockSparseMatrix(uniform_layout(num_blocks, size), uniform_layout(num_blocks, size))
    for i in range(num_blocks):
        for j in range(num_blocks):
            blk = A[i * size:(i + 1) * size, j * size:(j + 1) * size]
            if np.any(blk != 0.0):
                M.add_block(i, j, blk)
    return M, A


def test_pmg_full_separation_is_exact():
    M, A = random_block_spd(5, 3)
    b = np.random.default_rng(1).normal(size=A.shape[0])
    x = pmg_apply(M, b, 1, range(5), {}, dim=2)
    assert np.linalg.norm(b - A @ x) <= 1e-12 * np.linalg.norm(b)


def test_pmg_cache_reused():
    M, A = random_block_spd(4, 3)
    rng = np.random.default_rng(5)
    cache = {}
    pmg_apply(M, rng.normal(size=12), 0, range(4), cache, dim=2)
    stored = next(iter(cache.values()))
    pmg_apply(M, rng.normal(size=12), 0, range(4), cache, dim=2)
    assert len(cache) == 1 and next(iter(cache.values())) is stored


def test_pmg_partial_cell_set_supported_only_there():
    M, A = random_block_spd(4, 3, block_diagonal=True)
    b = np.random.default_rng(7).normal(size=12)
    x = pmg_apply(M, b, 0, (1, 2), {}, dim=2)
    assert np.all(x[:3] == 0.0) and np.all(x[9:] == 0.0) and np.any(x[3:9] != 0.0)


def test_pmg_decoupled_block_diagonal_exact():
    rng = np.random.default_rng(3)
    M = BlockSparseMatrix(uniform_layout(3, 3), uniform_layout(3, 3))
    A = np.zeros((9, 9))
    for c in range(3):
        B = np.zeros((3, 3))
        B[0, 0] = 1.0 + rng.random()
        H = rng.normal(size=(2, 2))
        B[1:, 1:] = H @ H.T + 2.0 * np.eye(2)
        M.add_block(c, c, B)
        A[3 * c:3 * c + 3, 3 * c:3 * c + 3] = B
    b = rng.normal(size=9)
    assert np.allclose(pmg_apply(M, b, 0, range(3), {}, dim=2),
                       np.linalg.solve(A, b), atol=1e-12)


def test_pmg_rejects_bad_cell_sets():
    M, _ = random_block_spd(3, 3)
    with pytest.raises(InvalidConfigError):
        pmg_apply(M, np.ones(9), 0, (), {}, dim=2)
    with pytest.raises(DimensionMismatchError):
        pmg_apply(M, np.ones(9), 0, (0, 7), {}, dim=2)


def test_pmg_singular_low_and_high_raise():
    M = BlockSparseMatrix(uniform_layout(3, 3), uniform_layout(3, 3))
    for c in (0, 2):
        M.add_block(c, c, np.eye(3))
    M.add_block(1, 1, np.zeros((3, 3)))
    with pytest.raises(SingularSystemError):
        pmg_apply(M, np.ones(9), 0, range(3), {}, dim=2)
    M2 = BlockSparseMatrix(uniform_layout(2, 3), uniform_layout(2, 3))
    M2.add_block(0, 0, np.eye(3))
    bad = np.zeros((3, 3))
    bad[0, 0] = 1.0
    M2.add_block(1, 1, bad)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        with pytest.raises(SingularSystemError):
            pmg_apply(M2, np.ones(6), 0, range(2), {}, dim=2)


def test_pmg_device_tensor_in_device_tensor_out():
    M, A = random_block_spd(4, 3)
    b = torch.randn(12, dtype=torch.float64, device="cuda")
    x = pmg_apply(M, b, 0, range(4), {}, dim=2)
    assert torch.is_tensor(x) and x.is_cuda
    xh = pmg_apply(M, b.cpu().numpy(), 0, range(4), {}, dim=2)
    assert np.array_equal(x.cpu().numpy(), xh)
