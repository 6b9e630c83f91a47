"""Stored-factorization direct solver on the device (drop-in for cutdg
`DirectFactorization` / `direct_factor` / `direct_apply`,
blockmatrix.py:203-243).

The reference factors with SuperLU (COLAMD + partial pivoting) and solves
on the host.  Here the matrix is assembled dense on the device
(xdg_pmg_build_low with every block), factored once by the hand-written
blocked partial-pivoting LU whose triangular factors are inverted in place
(xdg_batched_factor, csrc/xdg_factor.cu; setup), and every `apply` runs the
hand-written pivoted triangular-GEMV kernels (xdg_lu_inv_apply_*).  Dense storage bounds the size
(MAX_DENSE_DIRECT unknowns); the coarsest multigrid levels and the
low-order PMG systems it serves are small.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionMismatchError, SingularSystemError
from .factor import lu_inverse_dense

MAX_DENSE_DIRECT = 60000
F64 = torch.float64
I32 = torch.int32


def ipiv_to_perm(ctx, piv: torch.Tensor, dims: torch.Tensor,
                 vec_off: torch.Tensor) -> torch.Tensor:
    perm = torch.empty(piv.numel(), dtype=I32, device=ctx.device)
    nat.check(ctx.lib.xdg_ipiv_to_perm(int(dims.numel()), dims.data_ptr(),
                                       vec_off.data_ptr(), piv.data_ptr(),
                                       perm.data_ptr(), ctx.stream),
              "ipiv_to_perm")
    return perm


def dense_from_device_bsr(D) -> torch.Tensor:
    """Dense (n, n) device copy of a square DeviceBSR (all blocks)."""
    ctx = D.ctx
    n = D.nbr * D.N
    A = torch.zeros(n * n, dtype=F64, device=ctx.device)
    dev = ctx.device
    wi_ptr = D.row_ptr
    wi_blk = torch.arange(D.nnzb, dtype=I32, device=dev)
    wi_lrow = torch.arange(D.nbr, dtype=I32, device=dev)
    wi_sys = torch.zeros(D.nbr, dtype=I32, device=dev)
    lu_off = torch.zeros(1, dtype=torch.int64, device=dev)
    dims = torch.tensor([n], dtype=I32, device=dev)
    nat.check(ctx.lib.xdg_pmg_build_low(
        D.nbr, D.N, D.N, wi_ptr.data_ptr(), wi_blk.data_ptr(),
        D.col.data_ptr(), wi_lrow.data_ptr(), wi_sys.data_ptr(),
        lu_off.data_ptr(), dims.data_ptr(), D.val_t.data_ptr(), A.data_ptr(),
        ctx.stream), "pmg_build_low(dense)")
    return A.view(n, n)


class DeviceDirect:
    """Device-side factor of one dense system: apply(b_dev) -> x_dev."""

    def __init__(self, A: torch.Tensor, ctx, what="matrix"):
        n = A.shape[0]
        self.n = n
        self.ctx = ctx
        dev = ctx.device
        if n == 0:
            self.INV = torch.zeros(0, dtype=F64, device=dev)
            return
        # xdg_batched_factor: LU + triangular inverses in place (no library)
        self.INV, self.perm = lu_inverse_dense(ctx, A.contiguous(), what)
        self.lu_off = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dims = torch.tensor([n], dtype=I32, device=dev)
        self.row_sys = torch.zeros(n, dtype=I32, device=dev)
        self.scratch = torch.empty(2 * n, dtype=F64, device=dev)

    def apply(self, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.n, dtype=F64, device=b.device)
        if self.n == 0:
            return out
        nat.check(self.ctx.lib.xdg_lu_inv_apply(
            1, self.n, self.row_sys.data_ptr(), self.lu_off.data_ptr(),
            self.dims.data_ptr(), self.lu_off.data_ptr(), self.INV.data_ptr(),
            self.perm.data_ptr(), b.data_ptr(), out.data_ptr(),
            self.scratch.data_ptr(), self.ctx.stream), "lu_inv_apply")
        return out


# Above this many unknowns (uniform block layouts) the stored factorization
# is the multifrontal one (multifrontal.py).  A dense solve streams 8 n^2
# bytes in 3 launches, the multifrontal one far fewer bytes in ~5 launches
# per tree height: at n = 10,480 (cfg2 coarsest level) dense takes ~0.15 ms
# and multifrontal 0.25 ms (launch-bound), so dense stays up to here.
SPARSE_DIRECT_MIN = 16000


def _sparse_direct(M, n: int) -> bool:
    import os

    mode = os.environ.get("XDG_DIRECT", "auto")
    if M._padded_size() is not None or M.row_layout.num_blocks == 0:
        return False
    if mode in ("dense", "sparse"):
        return mode == "sparse"
    return n > SPARSE_DIRECT_MIN


class SparseDirect:
    """Device multifrontal factor of one square uniform-block DeviceBSR:
    apply(b_dev) -> x_dev (same interface as DeviceDirect)."""

    def __init__(self, D, ctx, what="matrix", comm=None):
        from .multifrontal import Multifrontal

        self.ctx = ctx
        self.n = D.nbr * D.N
        v = np.arange(D.nbr, dtype=np.int64) * D.N
        # comm (dist_solvers.Comm, world > 1): subtrees of the elimination
        # forest distributed over the ranks, top fronts replicated
        self.mf = Multifrontal(ctx, D.row_ptr.cpu().numpy(), D.col.cpu().numpy(), D.val_t,
                               D.N, [np.arange(D.nbr, dtype=np.int64)], D.N, v, v, what=what,
                               comm=comm)

    def apply(self, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.n, dtype=F64, device=b.device)
        return self.mf.solve(b, out)


class DirectFactorization:
    """Stored LU factorization reusable across right-hand sides
    (blockmatrix.py:203-227): `apply(b)` takes and returns numpy arrays;
    `apply_device` works on device tensors."""

    def __init__(self, matrix):
        from .blockmatrix import as_block_sparse
        from .device import Context

        M = as_block_sparse(matrix)
        self.shape = M.shape
        if self.shape[0] != self.shape[1]:
            raise DimensionMismatchError("direct solver needs a square matrix")
        n = self.shape[0]
        if _sparse_direct(M, n):
            from .device import Context

            ctx0 = Context.get()
            self._dev = SparseDirect(M.device(ctx0), ctx0)
            self.factor_count = 1
            return
        if n > MAX_DENSE_DIRECT:
            raise NotImplementedError(
                f"dense device LU limited to {MAX_DENSE_DIRECT} unknowns (got {n})")
        ctx = Context.get()
        if M._padded_size() is None and M.row_layout.num_blocks > 0:
            A = dense_from_device_bsr(M.device(ctx))
        else:
            A = torch.from_numpy(M.to_dense()).to(ctx.device)
        self._dev = DeviceDirect(A, ctx)
        del A
        self.factor_count = 1  # for reuse verification

    def apply_device(self, b: torch.Tensor, out=None) -> torch.Tensor:
        return self._dev.apply(b, out)

    def apply(self, b: np.ndarray) -> np.ndarray:
        b = np.asarray(b, dtype=float)
        if b.shape != (self.shape[0],):
            raise DimensionMismatchError(
                f"rhs of length {b.shape} against matrix {self.shape}")
        ctx = self._dev.ctx
        x = self._dev.apply(torch.from_numpy(b).to(ctx.device)).cpu().numpy()
        if not np.all(np.isfinite(x)):
            raise SingularSystemError("factorization produced non-finite values")
        return x


def direct_factor(M) -> DirectFactorization:
    return DirectFactorization(M)


def direct_apply(F: DirectFactorization, b: np.ndarray) -> np.ndarray:
    return F.apply(b)
