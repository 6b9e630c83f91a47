"""Drop-in for the transfer operations of the solver path
(cutdg transfer.py:344-351 galerkin_restrict, 408-453 containers).

`galerkin_restrict(M, b, R)` = (R^T M R, R^T b): the Galerkin coarse operator
(the paper's Table-2 "matrix-matrix" product).  The
symbolic phase (output pattern, per-output term lists) is vectorised on the
host; the numeric phase is the xdg_galerkin kernel (one CTA per coarse
block, terms R_i^T M_ik R_k accumulated in a fixed order).  R x_c and R^T r
of the solvers (solvers.py:730,734) are device BSR SpMVs.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .blockmatrix import BlockSparseMatrix, as_block_sparse
from .errors import LayoutMismatchError
from .hierarchy import HierarchyLevel, LevelInfo, MeshGraph, MultigridHierarchy  # noqa: F401

I32 = torch.int32


def galerkin_symbolic(rp, col, R_rp, R_col, n_coarse):
    """Pattern of R^T M R and its term lists.  Requires one R block per fine
    row.  Returns (Mc_row_ptr, Mc_col, tptr, t_e, t_ri, t_rk)."""
    rp, col = np.asarray(rp, np.int64), np.asarray(col, np.int64)
    R_rp, R_col = np.asarray(R_rp, np.int64), np.asarray(R_col, np.int64)
    if not np.all(np.diff(R_rp) == 1):
        raise LayoutMismatchError("Galerkin product expects one R block per fine row")
    parent = R_col
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    G, H = parent[rows], parent[col]
    order = np.lexsort((col, rows, H, G))          # (G, H, i, k)
    key = G[order] * n_coarse + H[order]
    first = np.flatnonzero(np.r_[True, key[1:] != key[:-1]]) if len(key) else np.zeros(0, np.int64)
    tptr = np.r_[first, len(key)]
    uk = key[first]
    c_rows, c_cols = uk // n_coarse, uk % n_coarse
    c_rp = np.zeros(n_coarse + 1, np.int64)
    np.cumsum(np.bincount(c_rows, minlength=n_coarse), out=c_rp[1:])
    return c_rp, c_cols, tptr, order, rows[order], col[order]


def galerkin_device(M, R):
    """Mc = R^T M R on the device.  M, R: BlockSparseMatrix (ours or the
    reference's); returns (DeviceBSR of Mc, host (row_ptr, col))."""
    from .device import Context, DeviceBSR

    M, R = as_block_sparse(M), as_block_sparse(R)
    ctx = Context.get()
    Md, Rd = M.device(ctx), R.device(ctx)
    if Md.N != Rd.N:
        raise LayoutMismatchError("M and R block sizes differ")
    nc = R.col_layout.num_blocks
    c_rp, c_col, tptr, te, tri, trk = galerkin_symbolic(
        Md.row_ptr.cpu().numpy(), Md.col.cpu().numpy(), Rd.row_ptr.cpu().numpy(),
        Rd.col.cpu().numpy(), nc)
    dev = ctx.device
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, I32)  # noqa: E731
    N = Md.N
    out = torch.empty(len(c_col), N, N, dtype=torch.float64, device=dev)
    targs = [up(tptr), up(te), up(tri), up(trk)]
    nat.check(ctx.lib.xdg_galerkin(len(c_col), N, *[t.data_ptr() for t in targs],
                                   Md.val_t.data_ptr(), Rd.val_t.data_ptr(),
                                   out.data_ptr(), ctx.stream), "galerkin")
    C = DeviceBSR(nc, nc, N, up(c_rp), up(c_col), out, ctx)
    return C, (c_rp, c_col)


def galerkin_restrict(M, b, R) -> tuple:
    """Coarse system (R^T M R, R^T b) (transfer.py:344-351)."""
    R = getattr(R, "matrix", R)
    Rb = as_block_sparse(R)
    C, (c_rp, c_col) = galerkin_device(M, Rb)
    rp, col, val = C.to_host_rowmajor()
    Mc = BlockSparseMatrix.from_bsr(c_rp, c_col, val, Rb.col_layout, Rb.col_layout)
    Mc._dev, Mc._dev_pad = C, None
    bc = None
    if b is not None:
        Rt = Rb.transpose()
        bc = Rt.matvec(np.asarray(b, dtype=float))
    return Mc, bc
