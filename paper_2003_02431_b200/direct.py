"""Stored-factorization direct solver on the device (drop-in for cutdg
`DirectFactorization` / `direct_factor` / `direct_apply`,
blockmatrix.py:203-243).

The reference factors with SuperLU (COLAMD + partial pivoting) and solves
on the host.  Here the matrix is assembled dense on the device
(xdg_pmg_build_low with every block), factored once with a partial-pivoting
LU (setup; torch.linalg.lu_factor_ex -> cuSOLVER getrf, plumbing), and every
`apply` runs the hand-written pivoted forward/backward substitution kernel
(xdg_lu_solve_batched).  Dense storage bounds the size
(MAX_DENSE_DIRECT unknowns); the coarsest multigrid levels and the
low-order PMG systems it serves are small.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionMismatchError, SingularSystemError

MAX_DENSE_DIRECT = 60000
F64 = torch.float64
I32 = torch.int32


def lu_factor_dense(A: torch.Tensor, what: str = "matrix"):
    """Partial-pivoting LU of one (n, n) or a batch (b, n, n) of dense
    device matrices.  Raises SingularSystemError on an exactly zero pivot or
    non-finite factor (SuperLU's 'Factor is exactly singular',
    blockmatrix.py:211-215; solvers.py:234-239)."""
    LU, piv, info = torch.linalg.lu_factor_ex(A)
    diag = torch.diagonal(LU, dim1=-2, dim2=-1)
    bad = (info != 0) | ~torch.isfinite(LU).flatten(-2).all(-1) | (diag == 0).any(-1)
    if bool(bad.any()):
        idx = torch.nonzero(bad.reshape(-1)).flatten()[:1].tolist()
        raise SingularSystemError(f"{what} is singular (system {idx})")
    return LU, piv


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


PANEL = 64          # rows per panel of xdg_lu_solve_panels
PANEL_MIN_N = 2048  # systems at least this large use the multi-CTA solve


class PanelFactor:
    """Extra setup for the multi-CTA solve of one large factored system:
    inverses of the 64x64 diagonal blocks of L (unit lower) and U."""

    def __init__(self, LU: torch.Tensor, ctx):
        n = LU.shape[0]
        self.n, self.ctx = n, ctx
        npan = (n + PANEL - 1) // PANEL
        pad = npan * PANEL - n
        dev = LU.device
        eye = torch.eye(PANEL, dtype=F64, device=dev)
        Lb = torch.empty(npan, PANEL, PANEL, dtype=F64, device=dev)
        Ub = torch.empty_like(Lb)
        for p in range(npan):
            r0, r1 = p * PANEL, min((p + 1) * PANEL, n)
            blk = eye.clone()
            blk[: r1 - r0, : r1 - r0] = LU[r0:r1, r0:r1]
            Lb[p] = torch.tril(blk, -1) + eye
            Ub[p] = torch.triu(blk)
            if r1 - r0 < PANEL:
                Ub[p, r1 - r0:, r1 - r0:] = eye[: pad, : pad]
        self.Linv = torch.linalg.solve_triangular(
            Lb, eye.expand_as(Lb), upper=False, unitriangular=True).contiguous()
        self.Uinv = torch.linalg.solve_triangular(
            Ub, eye.expand_as(Ub), upper=True).contiguous()
        self.counters = torch.zeros(4, dtype=I32, device=dev)

    def solve(self, LU_ptr: int, src_ptr: int, b: torch.Tensor, x_ptr: int):
        nat.check(self.ctx.lib.xdg_lu_solve_panels(
            self.n, LU_ptr, self.Linv.data_ptr(), self.Uinv.data_ptr(), src_ptr,
            b.data_ptr(), x_ptr, self.counters.data_ptr(), self.ctx.stream),
            "lu_solve_panels")


class DeviceDirect:
    """Device-side factor of one dense system: apply(b_dev) -> x_dev."""

    def __init__(self, A: torch.Tensor, ctx, what="matrix"):
        n = A.shape[0]
        self.n = n
        self.ctx = ctx
        dev = ctx.device
        if n == 0:
            self.LU = torch.zeros(0, dtype=F64, device=dev)
            return
        LU, piv = lu_factor_dense(A, what)
        self.LU = LU.contiguous()
        self.lu_off = torch.zeros(1, dtype=torch.int64, device=dev)
        self.vec_off = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dims = torch.tensor([n], dtype=I32, device=dev)
        self.perm = ipiv_to_perm(ctx, piv.to(I32).contiguous(), self.dims,
                                 self.vec_off)
        self.panel = PanelFactor(self.LU, ctx) if n >= PANEL_MIN_N else None

    def apply(self, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(self.n, dtype=F64, device=b.device)
        if self.n == 0:
            return out
        if self.panel is not None:
            self.panel.solve(self.LU.data_ptr(), self.perm.data_ptr(), b,
                             out.data_ptr())
            return out
        nat.check(self.ctx.lib.xdg_lu_solve_batched(
            1, self.lu_off.data_ptr(), self.dims.data_ptr(),
            self.vec_off.data_ptr(), self.LU.data_ptr(), self.perm.data_ptr(),
            b.data_ptr(), out.data_ptr(), self.ctx.stream), "lu_solve")
        return out


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
