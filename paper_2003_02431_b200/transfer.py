"""Drop-in for the transfer operations the solver path uses
(cutdg transfer.py:344-351 galerkin_restrict, 408-453 containers).

`galerkin_restrict` is setup (the paper's Table-2
"matrix-matrix" product); it runs on the host block SpGEMM of
blockmatrix.BlockSparseMatrix.matmat.  R x_c and R^T r (solvers.py:730,734)
are device BSR products inside the solvers.
"""
from __future__ import annotations

import numpy as np

from .blockmatrix import as_block_sparse, bs_matmat
from .hierarchy import HierarchyLevel, LevelInfo, MeshGraph, MultigridHierarchy  # noqa: F401


def galerkin_restrict(M, b, R) -> tuple:
    """Coarse system (R^T M R, R^T b)."""
    R = getattr(R, "matrix", R)
    M = as_block_sparse(M)
    R = as_block_sparse(R)
    Rt = R.transpose()
    Mc = bs_matmat(Rt, bs_matmat(M, R))
    bc = None if b is None else Rt.matvec(np.asarray(b, dtype=float))
    return Mc, bc
