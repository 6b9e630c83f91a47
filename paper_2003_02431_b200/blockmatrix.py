"""Drop-in `cutdg.blockmatrix` (reference: blockmatrix.py:1-255) whose
products run on the B200.

Host-side structure (dict of dense blocks keyed by (block-row, block-col),
additive `add_block`, layouts) keeps the reference's semantics; the
operations on the solver hot path -- `matvec` (blockmatrix.py:119-125) and
`DirectFactorization.apply` (blockmatrix.py:218-227) -- run through the
sm_100a C-ABI on a lazily built device mirror (`device()`), the analogue of
the reference's lazily cached CSR (blockmatrix.py:91-114).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np

from .errors import DimensionMismatchError, LayoutMismatchError


@dataclass(frozen=True)
class BlockLayout:
    """Sizes of the consecutive blocks of one axis (blockmatrix.py:26-49)."""

    sizes: tuple

    @property
    def offsets(self) -> np.ndarray:
        got = self.__dict__.get("_offsets")
        if got is None:
            got = np.zeros(len(self.sizes) + 1, dtype=np.int64)
            np.cumsum(np.asarray(self.sizes, dtype=np.int64), out=got[1:])
            object.__setattr__(self, "_offsets", got)
        return got

    @property
    def dim(self) -> int:
        return int(self.offsets[-1])

    @property
    def num_blocks(self) -> int:
        return len(self.sizes)

    def block_slice(self, b: int) -> slice:
        o = self.offsets
        return slice(int(o[b]), int(o[b + 1]))

    @property
    def uniform_size(self) -> Optional[int]:
        s = set(self.sizes)
        return s.pop() if len(s) == 1 else None


def uniform_layout(num_blocks: int, block_size: int) -> BlockLayout:
    return BlockLayout(sizes=(block_size,) * num_blocks)


class BlockSparseMatrix:
    """Block-sparse matrix with dense blocks (blockmatrix.py:56-200).

    Two ways in: the reference's incremental `add_block`, or
    :meth:`from_bsr` with (row_ptr, col, val) arrays for large operators
    (no per-block Python objects until `blocks` is touched).
    """

    def __init__(self, row_layout: BlockLayout, col_layout: BlockLayout):
        self.row_layout = row_layout
        self.col_layout = col_layout
        self._blocks: Optional[dict] = {}
        self._host_fn = None
        self._bsr = None  # (row_ptr, col, val) host arrays, sorted
        self._dev = None
        self._host_stream = None  # (HostStreamSpMV, pinned x, pinned y)

    @property
    def _bsr(self):
        if self._bsr_data is None and self._host_fn is not None:
            self._bsr_data, self._host_fn = self._host_fn(), None
        return self._bsr_data

    @_bsr.setter
    def _bsr(self, value):
        self._bsr_data = value

    # ---- construction ----------------------------------------------------
    @classmethod
    def from_bsr(cls, row_ptr, col, val, row_layout: BlockLayout,
                 col_layout: BlockLayout) -> "BlockSparseMatrix":
        M = cls(row_layout, col_layout)
        M._blocks = None
        M._bsr = (np.asarray(row_ptr, np.int64), np.asarray(col, np.int64),
                  np.asarray(val, np.float64))
        return M

    @classmethod
    def from_device(cls, dev, row_layout: BlockLayout,
                    col_layout: BlockLayout) -> "BlockSparseMatrix":
        """Wrap a DeviceBSR built in HBM (assembly, Galerkin products); the
        host arrays are copied back only if something asks for them."""
        M = cls(row_layout, col_layout)
        M._blocks = None
        M._host_fn = dev.to_host_rowmajor
        M._dev, M._dev_pad = dev, None
        return M

    @property
    def blocks(self) -> dict:
        if self._blocks is None:
            rp, col, val = self._bsr
            d = {}
            for bi in range(len(rp) - 1):
                for k in range(rp[bi], rp[bi + 1]):
                    d[(bi, int(col[k]))] = val[k]
            self._blocks = d
            self._bsr = None
        return self._blocks

    @property
    def shape(self) -> tuple:
        return (self.row_layout.dim, self.col_layout.dim)

    def add_block(self, bi: int, bj: int, block: np.ndarray) -> None:
        expected = (self.row_layout.sizes[bi], self.col_layout.sizes[bj])
        block = np.asarray(block)
        if block.shape != expected:
            raise DimensionMismatchError(
                f"block ({bi},{bj}) has shape {block.shape}, expected {expected}")
        blocks = self.blocks
        key = (bi, bj)
        if key in blocks:
            blocks[key] = blocks[key] + block
        else:
            blocks[key] = np.array(block, dtype=float)
        self._dev = None
        self._host_stream = None

    def get_block(self, bi: int, bj: int):
        if self._blocks is None:
            rp, col, val = self._bsr
            lo, hi = rp[bi], rp[bi + 1]
            k = lo + np.searchsorted(col[lo:hi], bj)
            if k < hi and col[k] == bj:
                return val[k]
            return None
        return self._blocks.get((bi, bj))

    @property
    def num_nonzero_blocks(self) -> int:
        if self._blocks is None:
            return len(self._bsr[1])
        return len(self._blocks)

    @property
    def nnz(self) -> int:
        if self._blocks is None:
            return int(self._bsr[2].size)
        return sum(b.size for b in self._blocks.values())

    # ---- sorted block arrays (tocsr order) -------------------------------
    def bsr_arrays(self, pad_to: Optional[int] = None):
        """(row_ptr, col, val[nnzb, n, n]) sorted by (bi, bj); blocks of a
        variable layout are zero-padded to `pad_to` (max block size)."""
        if self._blocks is None and pad_to is None:
            return self._bsr
        nbr = self.row_layout.num_blocks
        keys = sorted(self.blocks)
        N = pad_to or self.row_layout.uniform_size
        rp = np.zeros(nbr + 1, np.int64)
        if keys:
            np.add.at(rp, np.array([k[0] for k in keys]) + 1, 1)
        rp = np.cumsum(rp)
        col = np.array([k[1] for k in keys], np.int64)
        if pad_to is None:
            val = (np.stack([self.blocks[k] for k in keys]) if keys
                   else np.zeros((0, N, N)))
        else:
            val = np.zeros((len(keys), N, N))
            for i, k in enumerate(keys):
                b = self.blocks[k]
                val[i, : b.shape[0], : b.shape[1]] = b
        return rp, col, val

    def tocsr(self):
        """Host scipy CSR (export / tests), same construction order as the
        reference (blockmatrix.py:91-114)."""
        import scipy.sparse as sp

        ro, co = self.row_layout.offsets, self.col_layout.offsets
        rows, cols, vals = [], [], []
        for (bi, bj), block in sorted(self.blocks.items()):
            m, n = block.shape
            rows.append(np.repeat(np.arange(m) + ro[bi], n))
            cols.append(np.tile(np.arange(n) + co[bj], m))
            vals.append(block.ravel())
        if not rows:
            return sp.csr_matrix(self.shape)
        return sp.coo_matrix((np.concatenate(vals),
                              (np.concatenate(rows), np.concatenate(cols))),
                             shape=self.shape).tocsr()

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape)
        ro, co = self.row_layout.offsets, self.col_layout.offsets
        for (bi, bj), block in self.blocks.items():
            out[ro[bi]:ro[bi + 1], co[bj]:co[bj + 1]] += block
        return out

    # ---- device mirror ---------------------------------------------------
    def _padded_size(self) -> Optional[int]:
        n = self.row_layout.uniform_size
        if n is not None and n == self.col_layout.uniform_size:
            return None
        sizes = tuple(self.row_layout.sizes) + tuple(self.col_layout.sizes)
        return max(sizes) if sizes else 1

    def device(self, ctx=None):
        """Device mirror (DeviceBSR), built once and cached until the host
        blocks change.  Variable layouts are zero-padded to the largest
        block (padding adds exact zeros to every row sum)."""
        if self._dev is None:
            from .device import Context, DeviceBSR

            ctx = ctx or Context.get()
            pad = self._padded_size()
            rp, col, val = self.bsr_arrays(pad_to=pad)
            N = pad or self.row_layout.uniform_size
            if N is None:  # empty layouts
                N = 1
            self._dev = DeviceBSR.from_arrays(rp, col, val, N,
                                              self.col_layout.num_blocks, ctx)
            self._dev_pad = pad
        return self._dev

    def _pad_index(self, layout: BlockLayout, N: int) -> np.ndarray:
        """Positions of the layout's entries inside the padded vector."""
        sizes = np.asarray(layout.sizes, np.int64)
        starts = np.arange(len(sizes), dtype=np.int64) * N
        return np.concatenate([s + np.arange(n) for s, n in zip(starts, sizes)]) \
            if len(sizes) else np.zeros(0, np.int64)

    # host vectors above this many rows stream in z-slab chunks (transfers
    # overlapped with the SpMV); below, one chunk (fewest launches)
    STREAM_CHUNK_ROWS = 1 << 18

    def _host_streamer(self, D):
        """Cached HostStreamSpMV + pinned staging buffers of this matrix."""
        import torch

        from .device import HostStreamSpMV

        if self._host_stream is None or self._host_stream[0].D is not D:
            n = D.nbr * D.N
            # measured at cfg3 (22 M rows; profiles/r2_e2e_chunks.json): 8 / 12 /
            # 16 / 24 chunks -> 2,500 / 2,575 / 2,538 / 2,385 GB/s host to host
            chunks = (12 if n >= (1 << 22) else 8) if n >= self.STREAM_CHUNK_ROWS else 1
            self._host_stream = (HostStreamSpMV(D, chunks=chunks),
                                 torch.empty(n, dtype=torch.float64).pin_memory(),
                                 torch.empty(n, dtype=torch.float64).pin_memory())
        return self._host_stream

    def matvec(self, x, out=None):
        """y = M x on the GPU (blockmatrix.py:119-125); bit-identical to
        the reference's csr_matvec on tocsr().

        numpy in -> numpy out (the reference's contract): x is staged into
        pinned memory and the product streams host -> device -> host in
        row chunks, the transfers overlapped with the SpMV
        (device.HostStreamSpMV).  A pinned CPU torch tensor (optionally
        with a pinned `out`) skips the staging copies; a CUDA tensor stays
        on the device (CUDA in -> CUDA out)."""
        import torch

        if isinstance(x, torch.Tensor):
            xt = x.reshape(-1)
            if xt.numel() != self.shape[1] or xt.dtype != torch.float64:
                raise DimensionMismatchError(
                    f"vector of length {xt.numel()} ({xt.dtype}) against matrix {self.shape}")
        else:
            x = np.asarray(x, dtype=float)
            if x.shape != (self.shape[1],):
                raise DimensionMismatchError(
                    f"vector of length {x.shape} against matrix {self.shape}")
            xt = None
        if self.row_layout.num_blocks == 0:
            return np.zeros(0) if xt is None else torch.zeros(0, dtype=torch.float64,
                                                               device=xt.device)
        D = self.device()
        if self._dev_pad is not None:  # variable layouts: padded vectors
            N = self._dev_pad
            xv = xt.cpu().numpy() if xt is not None else x
            xp = np.zeros(self.col_layout.num_blocks * N)
            xp[self._pad_index(self.col_layout, N)] = xv
            y = D.spmv(torch.from_numpy(xp).to(D.ctx.device)).cpu().numpy()
            y = y[self._pad_index(self.row_layout, N)]
            return y if xt is None else torch.from_numpy(y).to(xt.device)
        if xt is not None and xt.is_cuda:
            return D.spmv(xt, out)
        if D.nbr != D.nbc:  # rectangular transfer operators: one staged product
            xd = (xt if xt is not None else torch.from_numpy(x)).to(D.ctx.device)
            y = D.spmv(xd).cpu()
            if out is not None:
                out.copy_(y)
                return out
            return y if xt is not None else y.numpy()
        hs, xh, yh = self._host_streamer(D)
        if xt is not None and xt.is_pinned():
            src = xt
        else:
            xh.copy_(xt if xt is not None else torch.from_numpy(x))
            src = xh
        dst = out if (out is not None and out.is_pinned()) else yh
        hs(src, dst, sync=True)  # blocks until dst holds the product
        if xt is None:
            return dst.numpy().copy() if out is None else out.copy_(dst)
        if out is not None:
            if dst is not out:
                out.copy_(dst)
            return out
        return dst.clone()

    def transpose(self) -> "BlockSparseMatrix":
        if self._blocks is None:  # array form: one stable sort, no dict
            rp, col, val = self._bsr
            rows = np.repeat(np.arange(len(rp) - 1, dtype=np.int64), np.diff(rp))
            o = np.lexsort((rows, col))
            trp = np.zeros(self.col_layout.num_blocks + 1, np.int64)
            np.cumsum(np.bincount(col, minlength=self.col_layout.num_blocks), out=trp[1:])
            return BlockSparseMatrix.from_bsr(
                trp, rows[o], np.ascontiguousarray(val[o].transpose(0, 2, 1)),
                self.col_layout, self.row_layout)
        out = BlockSparseMatrix(self.col_layout, self.row_layout)
        for (bi, bj), block in self.blocks.items():
            out.blocks[(bj, bi)] = block.T
        return out

    def matmat(self, other: "BlockSparseMatrix") -> "BlockSparseMatrix":
        """Block SpGEMM (setup; reference blockmatrix.py:133-151)."""
        if tuple(self.col_layout.sizes) != tuple(other.row_layout.sizes):
            raise LayoutMismatchError("inner block layouts do not match for matmat")
        out = BlockSparseMatrix(self.row_layout, other.col_layout)
        by_row: dict = {}
        for (bk, bj), block in other.blocks.items():
            by_row.setdefault(bk, []).append((bj, block))
        acc = out.blocks
        for (bi, bk), a_block in sorted(self.blocks.items()):
            for bj, b_block in by_row.get(bk, ()):
                prod = a_block @ b_block
                if (bi, bj) in acc:
                    acc[(bi, bj)] += prod
                else:
                    acc[(bi, bj)] = prod
        return out

    def extract_block_submatrix(self, row_blocks, col_blocks) -> "BlockSparseMatrix":
        rmap = {b: i for i, b in enumerate(row_blocks)}
        cmap = {b: i for i, b in enumerate(col_blocks)}
        out = BlockSparseMatrix(
            BlockLayout(tuple(self.row_layout.sizes[b] for b in row_blocks)),
            BlockLayout(tuple(self.col_layout.sizes[b] for b in col_blocks)))
        for (bi, bj), block in self.blocks.items():
            if bi in rmap and bj in cmap:
                out.blocks[(rmap[bi], cmap[bj])] = block
        return out

    def restrict_modes(self, row_modes: int, col_modes: int):
        import scipy.sparse as sp

        if self.row_layout.sizes and min(self.row_layout.sizes) < row_modes:
            raise DimensionMismatchError("row_modes exceeds a block size")
        if self.col_layout.sizes and min(self.col_layout.sizes) < col_modes:
            raise DimensionMismatchError("col_modes exceeds a block size")
        shape = (self.row_layout.num_blocks * row_modes,
                 self.col_layout.num_blocks * col_modes)
        keys = sorted(self.blocks)
        if not keys:
            return sp.csr_matrix(shape)
        r_idx = np.repeat(np.arange(row_modes), col_modes)
        c_idx = np.tile(np.arange(col_modes), row_modes)
        rows = np.concatenate([r_idx + bi * row_modes for bi, _ in keys])
        cols = np.concatenate([c_idx + bj * col_modes for _, bj in keys])
        vals = np.concatenate([self.blocks[k][:row_modes, :col_modes].ravel()
                               for k in keys])
        return sp.coo_matrix((vals, (rows, cols)), shape=shape).tocsr()

    def max_abs(self) -> float:
        if self._blocks is None:
            v = self._bsr[2]
            return float(np.max(np.abs(v))) if v.size else 0.0
        if not self._blocks:
            return 0.0
        return max(float(np.max(np.abs(b))) for b in self._blocks.values())


def bs_matvec(M: BlockSparseMatrix, x: np.ndarray) -> np.ndarray:
    return M.matvec(x)


def bs_matmat(A: BlockSparseMatrix, B: BlockSparseMatrix) -> BlockSparseMatrix:
    return A.matmat(B)


def as_block_sparse(M) -> BlockSparseMatrix:
    """Accept the reference's own BlockSparseMatrix (duck-typed: `.blocks`,
    `.row_layout`, `.col_layout`) as well as ours; reference objects get a
    cached device-capable twin (no copy of the numpy blocks)."""
    if isinstance(M, BlockSparseMatrix):
        return M
    twin = getattr(M, "_xdg_b200_twin", None)
    if twin is not None and twin[0] == len(M.blocks):
        return twin[1]
    out = BlockSparseMatrix(BlockLayout(tuple(M.row_layout.sizes)),
                            BlockLayout(tuple(M.col_layout.sizes)))
    out._blocks = dict(M.blocks)
    try:
        M._xdg_b200_twin = (len(M.blocks), out)
    except AttributeError:
        pass
    return out


def write_matrix_market(path, M: BlockSparseMatrix, comment: str = "") -> None:
    from scipy.io import mmwrite

    mmwrite(str(path), M.tocsr(), comment=comment)


def read_matrix_market(path):
    import scipy.sparse as sp
    from scipy.io import mmread

    return sp.csr_matrix(mmread(str(path)))


# DirectFactorization / direct_factor / direct_apply live in .direct (they
# need the dense LU kernels) and are re-exported here for API parity.
from .direct import DirectFactorization, direct_apply, direct_factor  # noqa: E402,F401
