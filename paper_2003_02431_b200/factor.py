"""Batched dense factorization through the sm_100a C-ABI (xdg_batched_factor,
csrc/xdg_factor.cu): partial-pivoting LU of many row-major matrices of any
sizes in place, optionally followed by their triangular inverses (the
layout the solve kernels xdg_lu_inv_apply* read).  Replaces the reference's
factorizations on the solver path -- SuperLU `splu` (cutdg
blockmatrix.py:203-216), `scipy.linalg.lu_factor` of the per-cell
high-order blocks (solvers.py:225-243) -- and the multifrontal fronts'
partial factorizations (multifrontal.py).  No library (cuSOLVER / MAGMA /
cuBLAS) call is involved.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import SingularSystemError

F64 = torch.float64
I32 = torch.int32
I64 = torch.int64

MAX_PER_CALL = 65535
WS_CAP_BYTES = 2 << 30


def batched_factor(ctx, A: torch.Tensor, off, n, p=None, ld=None, *, invert: bool,
                   perm: torch.Tensor | None = None, perm_off=None):
    """Factor matrix b (row-major, A[off[b]:], leading dimension ld[b],
    n[b] x n[b], first p[b] columns eliminated) for every b, in place.
    Returns (perm int32 device, perm_off int64 numpy, info int32 device):
    perm[perm_off[b] + i] = original row at position i (i < p[b]); info[b]
    != 0 marks a zero / non-finite pivot (see raise_if_singular)."""
    off = np.ascontiguousarray(off, np.int64)
    n = np.ascontiguousarray(n, np.int32)
    p = n.copy() if p is None else np.ascontiguousarray(p, np.int32)
    ld = n.copy() if ld is None else np.ascontiguousarray(ld, np.int32)
    nmat = len(off)
    dev = ctx.device
    if perm_off is None:
        perm_off = np.zeros(nmat, np.int64)
        np.cumsum(p[:-1], out=perm_off[1:])
    perm_off = np.ascontiguousarray(perm_off[:nmat], np.int64)
    need = int((perm_off + p).max()) if nmat else 0
    if perm is None:
        perm = torch.zeros(max(need, 1), dtype=I32, device=dev)
    elif perm.numel() < need:
        raise ValueError(f"perm buffer holds {perm.numel()} entries, {need} needed")
    info = torch.zeros(max(nmat, 1), dtype=I32, device=dev)
    if nmat == 0:
        return perm, perm_off, info
    lib = ctx.lib
    # calls of <= 65535 matrices whose sweep workspace stays bounded
    start = 0
    ws = None
    while start < nmat:
        stop = min(nmat, start + MAX_PER_CALL)
        if invert:
            while stop - start > 1:
                mp = int(p[start:stop].max())
                if lib.xdg_batched_factor_ws_bytes(stop - start, mp) <= WS_CAP_BYTES:
                    break
                stop = start + max(1, (stop - start) // 2)
        sl = slice(start, stop)
        max_n, max_p = int(n[sl].max()), int(p[sl].max())
        if invert:
            need = int(lib.xdg_batched_factor_ws_bytes(stop - start, max_p))
            if ws is None or ws.numel() * 8 < need:
                ws = torch.empty((need + 7) // 8, dtype=F64, device=dev)
        # the five descriptor arrays in ONE pinned, asynchronous upload (five
        # pageable copies per call each waited for the previous call's
        # kernels: 0.5 s of the cfg2 Schwarz multifrontal setup's 589 calls)
        k = stop - start
        desc = np.empty(2 * k + (3 * k + 1) // 2, np.int64)
        desc[:k] = off[sl]
        desc[k:2 * k] = perm_off[sl]
        i32 = desc[2 * k:].view(np.int32)
        i32[:k], i32[k:2 * k], i32[2 * k:3 * k] = n[sl], p[sl], ld[sl]
        d = torch.from_numpy(desc)
        if dev.type == "cuda":
            d = d.pin_memory().to(dev, non_blocking=True)
        base = d.data_ptr()
        nat.check(lib.xdg_batched_factor(
            k, base, base + 16 * k, base + 20 * k, base + 24 * k,
            max_n, max_p, A.data_ptr(), perm.data_ptr(), base + 8 * k,
            info[start:stop].data_ptr(), int(bool(invert)),
            ws.data_ptr() if ws is not None else None, ctx.stream), "batched_factor")
        del d  # stream-ordered: the caching allocators keep both buffers until the copy / kernels ran
        start = stop
    return perm, perm_off, info


def raise_if_singular(info: torch.Tensor, what: str, names=None) -> None:
    """SingularSystemError for the first matrix whose factorization met a
    zero pivot (SuperLU 'Factor is exactly singular', blockmatrix.py:211-215;
    lu_factor's singular warning promoted to an error, solvers.py:234-239)."""
    bad = torch.nonzero(info.reshape(-1))
    if bad.numel():
        i = int(bad[0])
        name = names(i) if callable(names) else i
        raise SingularSystemError(f"{what} is singular ({name})")


def lu_inverse_dense(ctx, A: torch.Tensor, what: str = "matrix"):
    """One dense contiguous (n, n) device matrix: LU + triangular inverses
    in place; returns (INV = A, perm)."""
    n = A.shape[0]
    if A.dim() != 2 or A.shape[1] != n or not A.is_contiguous():
        raise ValueError("lu_inverse_dense needs a contiguous (n, n) tensor")
    perm, _, info = batched_factor(ctx, A.view(-1), [0], [n], invert=True)
    raise_if_singular(info, what)
    return A, perm[:n]


def buckets_by_size(dims: np.ndarray):
    """Group systems of similar size (one xdg_batched_factor call each: the
    update grid is sized by the largest matrix of a call)."""
    dims = np.asarray(dims, np.int64)
    key = np.where(dims <= 64, (dims + 15) // 16, 4 + (dims + 127) // 128)
    for k in np.unique(key):
        yield np.flatnonzero(key == k)


def warmup(ctx) -> None:
    """Load the factorization kernels once (module loading, cluster launch
    attributes) outside a timed region -- the reference's LAPACK is likewise
    loaded before its solve timer starts."""
    n = 130
    A = torch.eye(n, dtype=F64, device=ctx.device)
    lu_inverse_dense(ctx, A)
    torch.cuda.synchronize(ctx.device)
