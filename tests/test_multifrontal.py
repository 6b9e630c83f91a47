"""Multifrontal sparse LU (multifrontal.py): nested-dissection forest,
numeric factorization on host tensors, solve checked through the numpy
restatement of the device kernels against dense solves.  The factorization
replaces SuperLU (cutdg blockmatrix.py:203-227); parity bar for exact
factorizations of the same system: <= 1e-10 relative."""
import numpy as np
import pytest
import torch

from mf_emulation import emulate_solve, front_factor_cpu
from paper_2003_02431_b200.errors import SingularSystemError
from paper_2003_02431_b200.multifrontal import Multifrontal, SystemGraph, nested_dissection


def grid_bsr(shape, N, seed=0, diag=8.0):
    """Block pattern of a Cartesian grid (face neighbours), random blocks
    with a dominant diagonal; returns (rp, col, vals row-major)."""
    rng = np.random.default_rng(seed)
    idx = np.arange(int(np.prod(shape))).reshape(shape)
    r, c = [idx.ravel()], [idx.ravel()]
    for ax in range(len(shape)):
        a = np.take(idx, range(shape[ax] - 1), axis=ax).ravel()
        b = np.take(idx, range(1, shape[ax]), axis=ax).ravel()
        r += [a, b]
        c += [b, a]
    r, c = np.concatenate(r), np.concatenate(c)
    o = np.lexsort((c, r))
    r, c = r[o], c[o]
    nb = idx.size
    rp = np.zeros(nb + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=nb), out=rp[1:])
    vals = 0.3 * rng.standard_normal((len(c), N, N))
    vals[r == c] += diag * np.eye(N)
    return rp, c, vals


def dense_sub(rp, col, vals, S, m):
    loc = {int(v): i for i, v in enumerate(S)}
    A = np.zeros((len(S) * m,) * 2)
    for i, v in enumerate(S):
        for k in range(rp[v], rp[v + 1]):
            j = loc.get(int(col[k]))
            if j is not None:
                A[i * m:(i + 1) * m, j * m:(j + 1) * m] = vals[k][:m, :m]
    return A


def build(rp, col, vals, N, sets, m, leaf=9):
    vsrc, vdst, off = [], [], 0
    for S in sets:
        vsrc.append(np.asarray(S) * N)
        vdst.append(off + np.arange(len(S)) * m)
        off += len(S) * m
    val_t = torch.from_numpy(np.ascontiguousarray(vals.transpose(0, 2, 1)))
    mf = Multifrontal(None, rp, col, val_t, N, sets, m, np.concatenate(vsrc),
                      np.concatenate(vdst), leaf_unknowns=leaf, front_factor=front_factor_cpu)
    return mf, off


@pytest.mark.parametrize("shape,N,m", [((9, 9), 4, 3), ((5, 4, 6), 3, 3), ((7,), 2, 2)])
def test_solve_matches_dense(shape, N, m):
    rp, col, vals = grid_bsr(shape, N)
    nb = len(rp) - 1
    rng = np.random.default_rng(1)
    sets = [np.arange(nb), np.sort(rng.choice(nb, nb // 3, replace=False)), np.array([nb - 1])]
    mf, xlen = build(rp, col, vals, N, sets, m)
    assert mf.nlevels >= 1
    b = rng.standard_normal(nb * N)
    x = emulate_solve(mf, b, xlen)
    off = 0
    for S in sets:
        A = dense_sub(rp, col, vals, S, m)
        ref = np.linalg.solve(A, b[(S[:, None] * N + np.arange(m)).reshape(-1)])
        got = x[off:off + len(ref)]
        assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)
        off += len(ref)


def test_pivoting_inside_fronts():
    """Zero leading diagonal entries force row exchanges inside the pivot
    blocks (partial pivoting, as SuperLU's)."""
    rp, col, vals = grid_bsr((6, 6), 3, seed=3)
    diag = np.flatnonzero(np.repeat(np.arange(len(rp) - 1), np.diff(rp)) == col)
    vals[diag, 0, 0] = 0.0
    vals[diag, 0, 1] = vals[diag, 1, 0] = 5.0
    mf, xlen = build(rp, col, vals, 3, [np.arange(36)], 3)
    b = np.random.default_rng(2).standard_normal(36 * 3)
    x = emulate_solve(mf, b, xlen)
    ref = np.linalg.solve(dense_sub(rp, col, vals, np.arange(36), 3), b)
    assert np.linalg.norm(x - ref) <= 1e-12 * np.linalg.norm(ref)


def test_singular_raises():
    rp, col, vals = grid_bsr((4, 4), 2)
    vals[:] = 0.0
    with pytest.raises(SingularSystemError):
        build(rp, col, vals, 2, [np.arange(16)], 2)


def test_nested_dissection_is_a_valid_elimination_forest():
    """Every vertex in exactly one front; no graph edge joins two fronts
    unless one is an ancestor of the other (separator property)."""
    rp, col, _ = grid_bsr((10, 10, 6), 1)
    G = SystemGraph(rp, col, [np.arange(600)])
    P, kids = nested_dissection(G.g_ptr, G.g_col, G.nv, 12)
    owner = np.full(G.nv, -1)
    for t, p in enumerate(P):
        assert (owner[p] == -1).all()
        owner[p] = t
    assert (owner >= 0).all()
    parent = np.full(len(P), -1)
    for t, ks in enumerate(kids):
        for c in ks:
            assert c < t  # post-order
            parent[c] = t

    def anc(a, b):  # is a an ancestor-or-self of b
        while b >= 0:
            if a == b:
                return True
            b = parent[b]
        return False

    rows = np.repeat(np.arange(G.nv), np.diff(G.g_ptr))
    for u, v in zip(rows, G.g_col):
        a, b = owner[u], owner[v]
        assert anc(a, b) or anc(b, a)


@pytest.mark.parametrize("shape,leaf,seed", [((10, 10, 6), 12, 0), ((17, 13), 5, 1),
                                              ((9, 9, 9), 30, 2)])
def test_native_ordering_matches_numpy_restatement(shape, leaf, seed):
    """xdg_nd_order / xdg_nd_boundaries (host C++) give exactly the fronts
    and boundary sets of the numpy restatement, incl. disconnected graphs."""
    from paper_2003_02431_b200.multifrontal import (
        boundaries,
        boundaries_py,
        nested_dissection_py,
    )

    rp, col, _ = grid_bsr(shape, 1, seed=seed)
    nb = len(rp) - 1
    rng = np.random.default_rng(seed)
    drop = rng.random(nb) < 0.08  # knock out vertices: several components
    keep = np.flatnonzero(~drop)
    sets = [keep[: len(keep) // 2], keep[len(keep) // 2:], np.array([0, 1, 2])]
    G = SystemGraph(rp, col, sets)
    P, kids = nested_dissection(G.g_ptr, G.g_col, G.nv, leaf)
    Pp, kp = nested_dissection_py(G.g_ptr, G.g_col, G.nv, leaf)
    assert len(P) == len(Pp) and kids == kp
    assert all(np.array_equal(a, b) for a, b in zip(P, Pp))
    owner = np.empty(G.nv, np.int64)
    for t, p in enumerate(P):
        owner[p] = t
    B = boundaries(G.g_ptr, G.g_col, G.nv, P, kids)
    Bp = boundaries_py(G.g_ptr, G.g_col, P, kids, owner)
    assert all(np.array_equal(a, b) for a, b in zip(B, Bp))


def test_native_ordering_many_components_threaded():
    """Hundreds of independent systems (Schwarz blocks): xdg_nd_order works on
    chunks of connected components in worker threads; the forest equals the
    numpy restatement's (one thread, component by component)."""
    from paper_2003_02431_b200.multifrontal import nested_dissection_py

    rp, col, _ = grid_bsr((24, 24), 1, seed=4)
    idx = np.arange(24 * 24).reshape(24, 24)
    sets = [np.sort(idx[max(i - 1, 0):i + 5, max(j - 1, 0):j + 5].ravel())
            for i in range(0, 24, 4) for j in range(0, 24, 4)] * 4  # 144 overlapping boxes
    G = SystemGraph(rp, col, sets)
    P, kids = nested_dissection(G.g_ptr, G.g_col, G.nv, 6)
    Pp, kp = nested_dissection_py(G.g_ptr, G.g_col, G.nv, 6)
    assert len(P) == len(Pp) and kids == kp
    assert all(np.array_equal(a, b) for a, b in zip(P, Pp))


def test_proportional_map_subtrees_and_shared_tops():
    """Subtree-to-rank mapping (multi-GPU factor): every front mapped;
    owned subtrees closed under children; a shared front has only shared or
    owned descendants and at least two ranks below it; world 1 owns all."""
    from paper_2003_02431_b200.multifrontal import proportional_map

    rp, col, _ = grid_bsr((12, 12, 6), 1)
    G = SystemGraph(rp, col, [np.arange(12 * 12 * 6)])
    P, kids = nested_dissection(G.g_ptr, G.g_col, G.nv, 8)
    nn = len(P)
    parent = np.full(nn, -1)
    for t, ks in enumerate(kids):
        for c in ks:
            parent[c] = t
    work = np.array([len(p) ** 2 for p in P], float)
    assert (proportional_map(kids, parent, work, 1) == 0).all()
    for world in (2, 3, 4, 8):
        r = proportional_map(kids, parent, work, world)
        assert set(np.unique(r[r >= 0])) == set(range(world))
        for t in range(nn):
            if r[t] >= 0:
                assert all(r[c] == r[t] for c in kids[t])
            else:
                below = set()
                stack = list(kids[t])
                while stack:
                    c = stack.pop()
                    if r[c] >= 0:
                        below.add(int(r[c]))
                    stack += kids[c]
                assert len(below) >= 2 or not kids[t]
        assert (r < 0).sum() < nn // 4  # only the top of the tree is replicated
