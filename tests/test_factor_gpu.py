"""Batched partial-pivoting LU + triangular inverses (xdg_batched_factor,
csrc/xdg_factor.cu) against numpy/scipy: the factorization the reference
gets from SuperLU / scipy lu_factor (blockmatrix.py:203-216,
solvers.py:225-243).  Reconstruction P A = L U, the pivot rule (LAPACK's
first maximal |a|), triangular inverses, multifrontal partial fronts
(Schur complement), singular detection, and the cluster path for large
matrices (panel rows in distributed shared memory)."""
import numpy as np
import pytest
import scipy.linalg as sla
import torch

from paper_2003_02431_b200.device import Context
from paper_2003_02431_b200.errors import SingularSystemError
from paper_2003_02431_b200.factor import batched_factor, lu_inverse_dense, raise_if_singular

pytestmark = pytest.mark.gpu


def _pack(mats):
    off = np.zeros(len(mats), np.int64)
    tot = 0
    for i, a in enumerate(mats):
        off[i] = tot
        tot += a.size
    flat = np.concatenate([a.ravel() for a in mats])
    return flat, off


def _split(flat, off, mats):
    return [flat[o:o + a.size].reshape(a.shape) for o, a in zip(off, mats)]


@pytest.mark.parametrize("invert", [False, True])
def test_batched_lu_variable_sizes(invert):
    ctx = Context.get()
    rng = np.random.default_rng(3)
    sizes = [1, 2, 5, 16, 31, 33, 64, 65, 100, 130, 257]
    mats = [rng.standard_normal((n, n)) for n in sizes]
    flat, off = _pack(mats)
    A = torch.from_numpy(flat).cuda()
    perm, poff, info = batched_factor(ctx, A, off, sizes, invert=invert)
    torch.cuda.synchronize()
    assert not info.any()
    out = _split(A.cpu().numpy(), off, mats)
    pm = perm.cpu().numpy()
    for a, f, po, n in zip(mats, out, poff, sizes):
        pr = pm[po:po + n]
        lu, piv = sla.lu_factor(a)
        sp = np.arange(n)
        for i, q in enumerate(piv):  # LAPACK ipiv -> permutation
            sp[[i, q]] = sp[[q, i]]
        assert np.array_equal(pr, sp), n  # same pivot rule as LAPACK getrf
        if invert:
            Li = np.tril(f, -1) + np.eye(n)
            Ui = np.triu(f)
            L = np.linalg.inv(Li)
            U = np.linalg.inv(Ui)
        else:
            L = np.tril(f, -1) + np.eye(n)
            U = np.triu(f)
            assert np.abs(f - lu).max() <= 1e-11 * max(1.0, np.abs(lu).max()), n
        r = np.abs(a[pr] - L @ U).max() / np.abs(a).max()
        assert r <= 1e-12 * max(n, 10), (n, r)


def test_partial_front_schur_complement():
    """n = P + B fronts, first P columns eliminated, pivots among the first
    P rows: L_BP, U_PB and the Schur complement F_BB - F_BP F_PP^-1 F_PB
    in place (the multifrontal front contract), with and without the
    triangular inverses of the pivot block."""
    ctx = Context.get()
    rng = np.random.default_rng(5)
    _check_partial_fronts([(10, 0), (10, 7), (40, 30), (64, 64), (100, 37), (150, 200)], 5)


@pytest.mark.parametrize("shape", [(96, 400), (300, 500), (200, 1500), (1280, 900), (416, 130)])
def test_partial_front_two_level_blocking(shape):
    """Fronts large enough for the super-panels (deferred trailing update,
    U12 block row by block row) and the 128 x 128 DMMA tiles."""
    _check_partial_fronts([shape], 11)


def test_mf_merge_products():
    """xdg_mf_merge: M = L_BP L^-1 and N = U^-1 U_PB of factored fronts
    against dense products (both tile sizes)."""
    import ctypes as C

    from paper_2003_02431_b200 import _native as nat

    ctx = Context.get()
    g = torch.Generator(device="cuda").manual_seed(7)
    for nb, P, B in [(3, 20, 50), (2, 96, 300), (2, 320, 130), (1, 700, 900)]:
        n = P + B
        Fb = torch.randn(nb, n, n, generator=g, dtype=torch.float64, device="cuda")
        M = torch.zeros(nb, B, P, dtype=torch.float64, device="cuda")
        N = torch.zeros(nb, P, B, dtype=torch.float64, device="cuda")
        nat.check(ctx.lib.xdg_mf_merge(nb, P, B, Fb.data_ptr(), M.data_ptr(), N.data_ptr(),
                                       ctx.stream), "mf_merge")
        INV = Fb[:, :P, :P]
        Li = torch.tril(INV, -1) + torch.eye(P, dtype=torch.float64, device="cuda")
        Mr = Fb[:, P:, :P] @ Li
        Nr = torch.triu(INV) @ Fb[:, :P, P:]
        assert float((M - Mr).abs().max() / Mr.abs().max()) <= 1e-13, (nb, P, B)
        assert float((N - Nr).abs().max() / Nr.abs().max()) <= 1e-13, (nb, P, B)


def _check_partial_fronts(shapes, seed):
    ctx = Context.get()
    rng = np.random.default_rng(seed)
    for invert in (False, True):
        mats = [rng.standard_normal((P + B, P + B)) for P, B in shapes]
        flat, off = _pack(mats)
        A = torch.from_numpy(flat).cuda()
        ns = [P + B for P, B in shapes]
        ps = [P for P, _ in shapes]
        perm, poff, info = batched_factor(ctx, A, off, ns, ps, invert=invert)
        assert not info.any()
        out = _split(A.cpu().numpy(), off, mats)
        pm = perm.cpu().numpy()
        for a, f, po, (P, B) in zip(mats, out, poff, shapes):
            pr = pm[po:po + P]
            FPP, FPB, FBP, FBB = a[:P, :P], a[:P, P:], a[P:, :P], a[P:, P:]
            if B:
                S = FBB - FBP @ np.linalg.solve(FPP, FPB)
                assert np.abs(f[P:, P:] - S).max() <= 1e-10 * max(1, np.abs(S).max()), (P, B)
            if invert:
                L = np.linalg.inv(np.tril(f[:P, :P], -1) + np.eye(P))
                U = np.linalg.inv(np.triu(f[:P, :P]))
            else:
                L, U = np.tril(f[:P, :P], -1) + np.eye(P), np.triu(f[:P, :P])
            assert np.abs(FPP[pr] - L @ U).max() <= 1e-11 * np.abs(FPP).max()
            if B:
                assert np.abs(f[P:, :P] @ U - FBP).max() <= 1e-10 * max(1, np.abs(FBP).max())
                assert np.abs(L @ f[:P, P:] - FPB[pr]).max() <= 1e-10 * max(1, np.abs(FPB).max())


@pytest.mark.parametrize("n", [700, 3000, 9000])
def test_large_dense_cluster_panel(n):
    """Large single matrices: the panel spans a cluster of up to 16 CTAs
    (distributed shared memory).  Backward error of the inverse-based solve
    x = U^-1 L^-1 P b, checked with device GEMMs (test infrastructure)."""
    ctx = Context.get()
    g = torch.Generator(device="cuda").manual_seed(n)
    A0 = torch.randn(n, n, generator=g, dtype=torch.float64, device="cuda")
    A0 += n ** 0.5 * torch.eye(n, dtype=torch.float64, device="cuda") * 0.1
    A = A0.clone()
    INV, perm = lu_inverse_dense(ctx, A)
    b = torch.randn(n, generator=g, dtype=torch.float64, device="cuda")
    Li = torch.tril(INV, -1) + torch.eye(n, dtype=torch.float64, device="cuda")
    Ui = torch.triu(INV)
    x = Ui @ (Li @ b[perm.long()])
    r = A0 @ x - b
    berr = float(r.abs().max() / (A0.abs().sum(1).max() * x.abs().max() + b.abs().max()))
    assert berr <= 1e-13, berr


def test_singular_detected():
    ctx = Context.get()
    rng = np.random.default_rng(1)
    a = rng.standard_normal((20, 20))
    a[:, 7] = 0.0
    b = rng.standard_normal((20, 20))
    flat, off = _pack([b, a])
    A = torch.from_numpy(flat).cuda()
    _, _, info = batched_factor(ctx, A, off, [20, 20], invert=True)
    inf = info.cpu().numpy()
    assert inf[0] == 0 and inf[1] == 8
    with pytest.raises(SingularSystemError):
        raise_if_singular(info, "test system")
