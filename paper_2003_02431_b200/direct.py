"""Stored-factorization direct solver on the device (drop-in for cutdg
`DirectFactorization` / `direct_factor` / `direct_apply`,
blockmatrix.py:203-243).

The reference factors with SuperLU (COLAMD + partial pivoting) and solves
on the host.  Here the matrix is assembled dense on the device
(xdg_pmg_build_low with every block), factored once with a partial-pivoting
LU (setup; torch.linalg.lu_factor_ex -> cuSOLVER getrf, plumbing) whose
triangular factors are inverted once (setup), and every `apply` runs the
hand-written pivoted triangular-GEMV kernels (xdg_lu_inv_apply_*).  Dense storage bounds the size
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


class _quiet_stdout:
    """Silence C-level stdout (MAGMA prints an advisory banner for batched
    getrf); flushes libc's buffer before restoring so nothing leaks into the
    one-line JSON contract of bench.py."""

    def __enter__(self):
        import ctypes
        import os
        import sys

        sys.stdout.flush()
        self._libc = ctypes.CDLL(None)
        self._libc.fflush(None)
        self._saved = os.dup(1)
        self._null = os.open(os.devnull, os.O_WRONLY)
        os.dup2(self._null, 1)
        return self

    def __exit__(self, *exc):
        import os

        self._libc.fflush(None)
        os.dup2(self._saved, 1)
        os.close(self._saved)
        os.close(self._null)


# Blocked batched LU for systems larger than LU_BLOCKED_MIN (XDG_LU_BLOCK =
# panel width, 0 = off).  tools/bench_lu_blocked.py on B200: 340 x 1920
# 0.293 s unblocked MAGMA vs 0.205 s blocked (nb 256); 1100 x 896 0.094 vs
# 0.096 s; 4400 x 448 0.059 vs 0.070 s.
LU_BLOCK = 256
LU_BLOCKED_MIN = 1280


def lu_factor_batched(A: torch.Tensor):
    """Partial-pivoting LU of a batch (b, n, n): MAGMA's batched getrf when
    the batch is large enough to pay off (5-17x faster per matrix than
    looping cuSOLVER at n = 512..1300, measured by tools/bench_setup_lu.py),
    cuSOLVER otherwise; large systems go through the right-looking blocked
    form (lu_factor_blocked: batched panel getrf + DGEMM trailing updates).
    Returns (LU, pivots, info)."""
    import os

    nb = int(os.environ.get("XDG_LU_BLOCK", LU_BLOCK))
    if A.dim() == 3 and A.shape[0] >= 4 and nb > 0 and A.shape[-1] > max(LU_BLOCKED_MIN, nb):
        return lu_factor_blocked(A, nb)
    return _lu_factor_unblocked(A)


def lu_factor_blocked(A: torch.Tensor, nb: int = LU_BLOCK):
    """Right-looking blocked LU with partial pivoting of a batch (b, n, n):
    per panel of nb columns, batched getrf of the (n-k) x nb panel (its
    pivots are the partial-pivoting choices over all remaining rows), the
    row swaps applied to the other columns (xdg_ipiv_to_perm + one gather),
    U12 = L11^-1 A12 (batched TRSM) and A22 -= L21 U12 (batched DGEMM).
    Same pivoting rule as unblocked getrf; roundoff-level differences only.
    Returns (LU, pivots (LAPACK 1-based), info) like lu_factor_ex."""
    from .device import Context

    ctx = Context.get()
    A = A.clone()
    b, n, _ = A.shape
    dev = A.device
    piv = torch.empty(b, n, dtype=torch.int32, device=dev)
    info = torch.zeros(b, dtype=torch.int32, device=dev)
    for k in range(0, n, nb):
        kb = min(nb, n - k)
        m = n - k
        LUp, pv, inf = _lu_factor_unblocked(A[:, k:, k:k + kb].contiguous())
        info = torch.where((info == 0) & (inf != 0), inf + k, info)
        pv = pv.to(torch.int32)
        piv[:, k:k + kb] = pv + k
        # sequential swaps of the panel -> permutation of the rows k..n-1
        ip = torch.arange(1, m + 1, dtype=torch.int32, device=dev).repeat(b, 1)
        ip[:, :kb] = pv
        dims = torch.full((b,), m, dtype=torch.int32, device=dev)
        off = torch.arange(b, dtype=torch.int64, device=dev) * m
        perm = ipiv_to_perm(ctx, ip.reshape(-1).contiguous(), dims, off).view(b, m).long()
        A[:, k:, :] = torch.gather(A[:, k:, :], 1, perm.unsqueeze(-1).expand(b, m, n))
        A[:, k:, k:k + kb] = LUp
        if k + kb < n:
            L11 = A[:, k:k + kb, k:k + kb]
            A[:, k:k + kb, k + kb:] = torch.linalg.solve_triangular(
                L11, A[:, k:k + kb, k + kb:], upper=False, unitriangular=True)
            A[:, k + kb:, k + kb:].baddbmm_(A[:, k + kb:, k:k + kb],
                                            A[:, k:k + kb, k + kb:], alpha=-1.0)
    return A, piv, info


def _lu_factor_unblocked(A: torch.Tensor):
    if A.dim() == 3 and A.shape[0] >= 4:
        prev = torch.backends.cuda.preferred_linalg_library()
        torch.backends.cuda.preferred_linalg_library("magma")
        try:
            with _quiet_stdout():
                out = torch.linalg.lu_factor_ex(A)
                torch.cuda.synchronize(A.device)
        finally:
            torch.backends.cuda.preferred_linalg_library(prev)
        return out
    return torch.linalg.lu_factor_ex(A)


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


def triangular_inverses(LU: torch.Tensor, chunk_bytes: int = 2 << 30) -> torch.Tensor:
    """INV of a packed LU (n, n) or batch (b, n, n): L^-1 strictly below the
    diagonal (unit diagonal implicit), U^-1 on and above it (setup; the
    inverses of triangular matrices via torch.linalg.solve_triangular)."""
    if LU.dim() == 2:
        return triangular_inverses(LU.unsqueeze(0), chunk_bytes)[0]
    nb, n, _ = LU.shape
    out = torch.empty_like(LU)
    eye = torch.eye(n, dtype=LU.dtype, device=LU.device)
    step = max(1, chunk_bytes // max(1, 8 * n * n * 4))
    for s in range(0, nb, step):
        blk = LU[s:s + step]
        Linv = torch.linalg.solve_triangular(torch.tril(blk, -1) + eye, eye.expand_as(blk),
                                             upper=False, unitriangular=True)
        Uinv = torch.linalg.solve_triangular(torch.triu(blk), eye.expand_as(blk),
                                             upper=True)
        out[s:s + step] = torch.tril(Linv, -1) + torch.triu(Uinv)
    return out


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
        LU, piv = lu_factor_dense(A, what)
        self.INV = triangular_inverses(LU).contiguous()
        del LU
        self.lu_off = torch.zeros(1, dtype=torch.int64, device=dev)
        self.dims = torch.tensor([n], dtype=I32, device=dev)
        self.perm = ipiv_to_perm(ctx, piv.to(I32).contiguous(), self.dims, self.lu_off)
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

    def __init__(self, D, ctx, what="matrix"):
        from .multifrontal import Multifrontal

        self.ctx = ctx
        self.n = D.nbr * D.N
        v = np.arange(D.nbr, dtype=np.int64) * D.N
        self.mf = Multifrontal(ctx, D.row_ptr.cpu().numpy(), D.col.cpu().numpy(), D.val_t,
                               D.N, [np.arange(D.nbr, dtype=np.int64)], D.N, v, v, what=what)

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
