"""Blocked batched LU (direct.lu_factor_blocked: panel getrf + TRSM +
DGEMM updates) vs the unblocked batched getrf it replaces for large
systems: same partial-pivoting rule, P L U = A to roundoff, same solves."""
import pytest
import torch

from paper_2003_02431_b200.direct import _lu_factor_unblocked, lu_factor_blocked

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("b,n,nb", [(4, 300, 64), (6, 517, 128), (5, 256, 128)])
def test_blocked_lu_matches_unblocked(b, n, nb):
    g = torch.Generator(device="cuda").manual_seed(n)
    A = torch.randn(b, n, n, dtype=torch.float64, device="cuda", generator=g)
    A[:, torch.arange(n), torch.arange(n)] *= 0.01  # force pivoting
    LU, piv, info = lu_factor_blocked(A, nb)
    LU0, piv0, info0 = _lu_factor_unblocked(A)
    assert int(info.abs().sum()) == 0 and int(info0.abs().sum()) == 0
    P, L, U = torch.lu_unpack(LU, piv)
    rec = (P @ L @ U - A).flatten(1).norm(dim=1) / A.flatten(1).norm(dim=1)
    assert float(rec.max()) <= 1e-13
    # partial pivoting picks the same rows (no near-ties in random data)
    assert torch.equal(piv.to(torch.int64), piv0.to(torch.int64))
    rhs = torch.randn(b, n, 1, dtype=torch.float64, device="cuda", generator=g)
    x = torch.linalg.lu_solve(LU, piv, rhs)
    x0 = torch.linalg.lu_solve(LU0, piv0, rhs)
    assert float(((x - x0).norm() / x0.norm())) <= 1e-11


def test_blocked_lu_reports_singular():
    A = torch.randn(4, 300, 300, dtype=torch.float64, device="cuda")
    A[2, :, 150] = 0.0  # a zero column: zero pivot at step 151
    _, _, info = lu_factor_blocked(A, 64)
    assert int(info[2]) > 0 and int(info[[0, 1, 3]].abs().sum()) == 0
