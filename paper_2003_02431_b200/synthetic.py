"""BASELINE config 3: synthetic block-MSR operator on a 3D Cartesian grid
(128^3 cells, p=2 -> N=10, 7-point cell stencil, 5 % cut cells carrying a
second species block).  Pattern recipe: SURVEY.md 8(d) "Exact recipes".

Block rows follow the reference's index-map order (spaces.py:80-85): cells
ascending (x fastest), species A before species B of a cut cell.  Pattern:
(A,A) for every cell; (B,B), (A,B), (B,A) inside cut cells; for each of the
6 face neighbours a->b: (A_a, A_b), and (B_a, B_b) when both cells are cut.

`cfg3_pattern` is the vectorised pattern (int64 numpy).  `cfg3_slab_device`
builds the rows of a contiguous z-slab directly in HBM with seeded device
random values of the recipe's distributions (diagonal A^T A + 10 I with
A ~ N(0,1), off-diagonal 0.1 N(0,1)); the exact numpy value stream of the
recipe lives in oracle/cfg3.py (test infrastructure) and is used for parity
at sizes the CPU can build.
"""
from __future__ import annotations

import numpy as np
import torch


def cut_mask(n: int, seed: int = 0, frac: float = 0.05) -> np.ndarray:
    J = n ** 3
    rng = np.random.default_rng(seed)
    cut = np.zeros(J, bool)
    cut[rng.choice(J, size=int(round(frac * J)), replace=False)] = True
    return cut


def block_rows_of(cut: np.ndarray) -> np.ndarray:
    """first[j]: block row of species A of cell j (B is first[j] + 1)."""
    first = np.zeros(len(cut) + 1, np.int64)
    np.cumsum(1 + cut.astype(np.int64), out=first[1:])
    return first


def _neighbour_pairs(n: int, cells: np.ndarray):
    """(a, b) for every in-range face neighbour b of a, a in `cells`."""
    x = cells % n
    y = (cells // n) % n
    z = cells // (n * n)
    A, B = [], []
    for coord, stride in ((x, 1), (y, n), (z, n * n)):
        for sgn in (-1, 1):
            ok = (coord + sgn >= 0) & (coord + sgn < n)
            A.append(cells[ok])
            B.append(cells[ok] + sgn * stride)
    return np.concatenate(A), np.concatenate(B)


def cfg3_pattern(n: int, seed: int = 0, cells: np.ndarray | None = None,
                 cut: np.ndarray | None = None):
    """Sorted block pattern of the rows of `cells` (default: all cells).

    Returns (rows, cols, is_diag, first, cut) with rows/cols GLOBAL block
    indices sorted by (row, col).
    """
    if cut is None:
        cut = cut_mask(n, seed)
    first = block_rows_of(cut)
    if cells is None:
        cells = np.arange(n ** 3, dtype=np.int64)
    fc = first[cells]
    cc = cut[cells]
    rows = [fc, fc[cc] + 1, fc[cc], fc[cc] + 1]
    cols = [fc, fc[cc] + 1, fc[cc] + 1, fc[cc]]
    a, b = _neighbour_pairs(n, cells)
    rows.append(first[a])
    cols.append(first[b])
    both = cut[a] & cut[b]
    rows.append(first[a[both]] + 1)
    cols.append(first[b[both]] + 1)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    return rows, cols, rows == cols, first, cut


def cfg3_counts(n: int, seed: int = 0) -> tuple:
    rows, cols, _, first, cut = cfg3_pattern(n, seed)
    return int(first[-1]), int(len(rows))


def slab_cells(n: int, rank: int, world: int) -> np.ndarray:
    """Cells of the contiguous z-slab of `rank` (z planes split evenly)."""
    z0 = (n * rank) // world
    z1 = (n * (rank + 1)) // world
    return np.arange(z0 * n * n, z1 * n * n, dtype=np.int64)


def cfg3_slab_host(n: int, rank: int = 0, world: int = 1, seed: int = 0,
                   cut: np.ndarray | None = None) -> dict:
    """Host pattern of one z-slab: local row_ptr, local columns renumbered
    [owned | ghosts (sorted global ids)], the slab's global block-row range,
    the ghost ids and the global block indices of the local blocks (the
    local blocks keep the global (row, col) storage order, so per-row sums
    run in the reference's order)."""
    if cut is None:
        cut = cut_mask(n, seed)
    first = block_rows_of(cut)
    cells = slab_cells(n, rank, world)
    rows, cols, is_diag, _, _ = cfg3_pattern(n, seed, cells=cells, cut=cut)
    row0 = int(first[cells[0]]) if len(cells) else 0
    row1 = int(first[cells[-1] + 1]) if len(cells) else 0
    nloc = row1 - row0
    ghosts = np.unique(cols[(cols < row0) | (cols >= row1)])
    owned = (cols >= row0) & (cols < row1)
    lcol = np.where(owned, cols - row0, 0)
    lcol[~owned] = nloc + np.searchsorted(ghosts, cols[~owned])
    rp = np.zeros(nloc + 1, np.int64)
    np.cumsum(np.bincount(rows - row0, minlength=nloc), out=rp[1:])
    # global block index of every local block (global storage is sorted by
    # (row, col) too, and the slab's rows are contiguous)
    nnz_before = 0
    if row0 > 0:
        r_all, _, _, _, _ = cfg3_pattern(n, seed, cells=np.arange(cells[0]), cut=cut) \
            if cells[0] > 0 else (np.zeros(0), None, None, None, None)
        nnz_before = len(r_all)
    ks = nnz_before + np.arange(len(rows), dtype=np.int64)
    return dict(row_ptr=rp, col=lcol, is_diag=is_diag, row0=row0, row1=row1,
                ghosts=ghosts, halo_lo=ghosts[ghosts < row0],
                halo_hi=ghosts[ghosts >= row1], global_blocks=ks,
                nbr_global=int(first[-1]), cut=cut, first=first)


def cfg3_slab_device(n: int, rank: int = 0, world: int = 1, seed: int = 0,
                     N: int = 10, ctx=None, value_seed: int = 1234):
    """Local operator of one z-slab, built in HBM.

    Returns the cfg3_slab_host dict plus D = DeviceBSR over the local rows
    (columns [owned blocks | halo blocks]) and L_global.  Values are seeded
    device random numbers with the recipe's distributions (diagonal
    A^T A + 10 I, A ~ N(0,1); off-diagonal 0.1 N(0,1)).
    """
    from .device import Context, DeviceBSR

    ctx = ctx or Context.get()
    dev = ctx.device
    h = cfg3_slab_host(n, rank, world, seed)
    rp, lcol, is_diag = h["row_ptr"], h["col"], h["is_diag"]
    nloc = h["row1"] - h["row0"]
    nnzb = len(lcol)
    g = torch.Generator(device=dev)
    g.manual_seed(value_seed + rank)
    val = torch.empty(nnzb, N, N, dtype=torch.float64, device=dev)
    diag_idx = torch.from_numpy(np.flatnonzero(is_diag)).to(dev)
    off_idx = torch.from_numpy(np.flatnonzero(~is_diag)).to(dev)
    chunk = 1 << 20
    for s in range(0, len(off_idx), chunk):
        idx = off_idx[s:s + chunk]
        val[idx] = 0.1 * torch.randn(len(idx), N, N, generator=g, device=dev,
                                     dtype=torch.float64)
    eye = 10.0 * torch.eye(N, dtype=torch.float64, device=dev)
    for s in range(0, len(diag_idx), chunk):
        idx = diag_idx[s:s + chunk]
        A = torch.randn(len(idx), N, N, generator=g, device=dev, dtype=torch.float64)
        # A^T A as N rank-one updates in k order (elementwise kernels: no
        # library GEMM appears in the bench process's launch list)
        G = eye.expand(len(idx), N, N).clone()
        for k in range(N):
            G.addcmul_(A[:, k, :, None], A[:, k, None, :])
        val[idx] = G
    # random blocks are layout-agnostic and A^T A + 10 I is symmetric, so the
    # values are written directly as column-major blocks
    h["D"] = DeviceBSR.from_arrays(rp, lcol, val, N, nloc + len(h["ghosts"]), ctx,
                                   val_is_colmajor=True)
    h["L_global"] = h["nbr_global"] * N
    return h
