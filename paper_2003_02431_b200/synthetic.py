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


def cfg3_slab_device(n: int, rank: int = 0, world: int = 1, seed: int = 0,
                     N: int = 10, ctx=None, value_seed: int = 1234):
    """Local operator of one z-slab, built in HBM.

    Returns dict(D=DeviceBSR over local rows with columns renumbered to
    [owned blocks | halo blocks], row0/row1 = global block-row range,
    halo_lo/halo_hi = global block rows of the ghost planes (below/above),
    L_global, nbr_global, nnzb_global).
    """
    from .device import Context, DeviceBSR

    ctx = ctx or Context.get()
    dev = ctx.device
    cut = cut_mask(n, seed)
    first = block_rows_of(cut)
    cells = slab_cells(n, rank, world)
    rows, cols, is_diag, _, _ = cfg3_pattern(n, seed, cells=cells, cut=cut)
    row0 = int(first[cells[0]]) if len(cells) else 0
    row1 = int(first[cells[-1] + 1]) if len(cells) else 0
    nloc = row1 - row0
    # halo: global block rows of the neighbouring z planes that appear as cols
    ghost = np.unique(cols[(cols < row0) | (cols >= row1)])
    lo = ghost[ghost < row0]
    hi = ghost[ghost >= row1]
    # local column numbering: owned [0, nloc), ghosts after (lo then hi)
    gmap_keys = np.concatenate([lo, hi])
    lcol = np.where((cols >= row0) & (cols < row1), cols - row0, -1)
    gpos = np.searchsorted(gmap_keys, cols[lcol < 0])
    lcol[lcol < 0] = nloc + gpos
    lrow = rows - row0
    rp = np.zeros(nloc + 1, np.int64)
    np.cumsum(np.bincount(lrow, minlength=nloc), out=rp[1:])
    nnzb = len(rows)
    # values on the device, generated directly column-major (the generator
    # fills the block; the diagonal A^T A + 10 I is symmetric anyway)
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
        val[idx] = torch.bmm(A.transpose(1, 2), A) + eye
    D = DeviceBSR.from_arrays(rp, lcol, val, N, nloc + len(gmap_keys), ctx,
                              val_is_colmajor=True)
    return dict(D=D, row0=row0, row1=row1, halo_lo=lo, halo_hi=hi,
                L_global=int(first[-1]) * N, nbr_global=int(first[-1]),
                cut=cut, first=first)
