"""Device-resident objects of the hot path: the BSR-T matrix mirror and the
vector kernels, over torch CUDA storage (torch is plumbing here: device
memory and the stream; every FLOP runs in libxdg_b200.so).

`DeviceBSR` is the device mirror of a uniform-block BlockSparseMatrix
(cutdg blockmatrix.py:56-200): row_ptr/col int32, blocks f64 column-major.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import DimensionMismatchError, NativeLibraryError

F64 = torch.float64


def _ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


class Context:
    """Per-process device context: the CUDA device, the stream the kernels
    run on, and the reduction workspaces (one per stream)."""

    _instances: dict = {}

    def __init__(self, device: torch.device):
        self.device = device
        self.lib = nat.load()
        with torch.cuda.device(device):
            nb = int(self.lib.xdg_reduce_workspace_bytes())
            self._ws = torch.zeros((nb + 7) // 8, dtype=F64, device=device)
            self._gemv_ws = torch.zeros(1, dtype=F64, device=device)
            self._scalars = torch.zeros(64, dtype=F64, device=device)

    @classmethod
    def get(cls, device=None) -> "Context":
        if not torch.cuda.is_available():
            raise NativeLibraryError(
                "no CUDA device: the xdg_b200 solver path has no CPU fallback")
        dev = torch.device(device if device is not None else "cuda",
                           ) if not isinstance(device, torch.device) else device
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        ctx = cls._instances.get(dev)
        if ctx is None:
            ctx = cls(dev)
            cls._instances[dev] = ctx
        return ctx

    @property
    def stream(self) -> int:
        return torch.cuda.current_stream(self.device).cuda_stream

    @property
    def ws(self) -> int:
        return self._ws.data_ptr()

    def gemv_ws(self, ncols: int) -> int:
        need = (int(self.lib.xdg_gemv_t_workspace_bytes(max(ncols, 1))) + 7) // 8
        if self._gemv_ws.numel() < need:
            self._gemv_ws = torch.zeros(need, dtype=F64, device=self.device)
        return self._gemv_ws.data_ptr()

    # ---- vector kernels -------------------------------------------------
    def dot(self, x: torch.Tensor, y: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
        nat.check(self.lib.xdg_dot(x.numel(), x.data_ptr(), y.data_ptr(),
                                   out.data_ptr(), self.ws, self.stream), "dot")
        return out

    def axpy(self, a: float, x, y, a_dev=None):
        nat.check(self.lib.xdg_axpy(y.numel(), float(a), _ptr(a_dev),
                                    x.data_ptr(), y.data_ptr(), self.stream),
                  "axpy")
        return y

    def scale(self, a: float, x, y, a_dev=None, invert=False):
        nat.check(self.lib.xdg_scale(y.numel(), float(a), _ptr(a_dev),
                                     int(bool(invert)), x.data_ptr(),
                                     y.data_ptr(), self.stream), "scale")
        return y

    def sub(self, b, y, r):
        nat.check(self.lib.xdg_sub(r.numel(), b.data_ptr(), y.data_ptr(),
                                   r.data_ptr(), self.stream), "sub")
        return r

    def div(self, x, d, y):
        nat.check(self.lib.xdg_div(y.numel(), x.data_ptr(), d.data_ptr(),
                                   y.data_ptr(), self.stream), "div")
        return y

    def gemv_t(self, W, ncols: int, w, coeff):
        L = w.numel()
        ld = W.stride(0) if W.dim() == 2 else L
        nat.check(self.lib.xdg_gemv_t(L, int(ncols), W.data_ptr(), ld,
                                      w.data_ptr(), coeff.data_ptr(),
                                      self.gemv_ws(ncols), self.stream),
                  "gemv_t")
        return coeff

    def gemv_update2(self, W, Z, ncols: int, coeff, w, z):
        L = w.numel()
        ld = W.stride(0)
        nat.check(self.lib.xdg_gemv_update2(
            L, int(ncols), W.data_ptr(), _ptr(Z), ld, coeff.data_ptr(), None,
            w.data_ptr(), _ptr(z), self.stream), "gemv_update2")


class DeviceBSR:
    """Uniform-block BSR matrix resident in HBM, blocks column-major.

    Built from the reference's row-major block arrays (tocsr order,
    blockmatrix.py:91-114); the row-major -> column-major conversion runs on
    the device (xdg_blocks_transpose).
    """

    def __init__(self, nbr: int, nbc: int, N: int, row_ptr: torch.Tensor,
                 col: torch.Tensor, val_t: torch.Tensor, ctx: Context):
        self.nbr, self.nbc, self.N = int(nbr), int(nbc), int(N)
        self.row_ptr, self.col, self.val_t = row_ptr, col, val_t
        self.ctx = ctx
        self.nnzb = int(col.numel())

    @property
    def shape(self):
        return (self.nbr * self.N, self.nbc * self.N)

    @classmethod
    def from_arrays(cls, row_ptr, col, val, N: int, nbc: int,
                    ctx: Context | None = None, val_is_colmajor=False):
        """row_ptr/col: integer arrays (numpy or torch), val: (nnzb, N, N)
        row-major blocks (numpy or torch, host or device)."""
        ctx = ctx or Context.get()
        dev = ctx.device
        rp = torch.as_tensor(np.asarray(row_ptr) if not torch.is_tensor(row_ptr)
                             else row_ptr).to(device=dev, dtype=torch.int32)
        cl = torch.as_tensor(np.asarray(col) if not torch.is_tensor(col)
                             else col).to(device=dev, dtype=torch.int32)
        nbr = rp.numel() - 1
        nnzb = cl.numel()
        if torch.is_tensor(val):
            v = val.to(device=dev, dtype=F64).reshape(nnzb, N, N).contiguous()
        else:
            v = torch.from_numpy(np.ascontiguousarray(val, dtype=np.float64)
                                 .reshape(nnzb, N, N)).to(dev)
        if val_is_colmajor:
            vt = v
        else:
            vt = torch.empty_like(v)
            nat.check(ctx.lib.xdg_blocks_transpose(nnzb, N, v.data_ptr(),
                                                   vt.data_ptr(), ctx.stream),
                      "blocks_transpose")
            del v
        return cls(nbr, nbc, N, rp, cl, vt, ctx)

    def spmv(self, x: torch.Tensor, y: torch.Tensor | None = None, *,
             alpha: float = 1.0, beta: float = 0.0, b: torch.Tensor | None = None,
             norm_out: torch.Tensor | None = None, rows=None) -> torch.Tensor:
        """y = alpha M x + beta y, or y = b - M x when b is given; optional
        fused ||y||^2 into the device scalar norm_out."""
        if x.numel() < self.nbc * self.N:
            raise DimensionMismatchError(
                f"vector of length {x.numel()} against matrix {self.shape}")
        if y is None:
            y = torch.empty(self.nbr * self.N, dtype=F64, device=x.device)
        rb, re = (0, self.nbr) if rows is None else rows
        nat.check(self.ctx.lib.xdg_bsr_spmv(
            rb, re, self.N, self.row_ptr.data_ptr(), self.col.data_ptr(),
            self.val_t.data_ptr(), x.data_ptr(), y.data_ptr(), float(alpha),
            float(beta), _ptr(b), _ptr(norm_out), self.ctx.ws,
            self.ctx.stream), "bsr_spmv")
        return y

    def algorithmic_bytes(self, fused_b: bool = False) -> int:
        """8 N^2 nnzb + 4 nnzb + 4 (nbr+1) + 8 L_x + 8 L_y."""
        N = self.N
        b = (8 * N * N * self.nnzb + 4 * self.nnzb + 4 * (self.nbr + 1)
             + 8 * self.nbc * N + 8 * self.nbr * N)
        return b + (8 * self.nbr * N if fused_b else 0)

    def flops(self) -> int:
        return 2 * self.N * self.N * self.nnzb

    def to_host_rowmajor(self) -> tuple:
        """(row_ptr, col, val[nnzb,N,N] row-major) as numpy (tests)."""
        v = torch.empty_like(self.val_t)
        nat.check(self.ctx.lib.xdg_blocks_transpose(
            self.nnzb, self.N, self.val_t.data_ptr(), v.data_ptr(),
            self.ctx.stream), "blocks_transpose")
        return (self.row_ptr.cpu().numpy().astype(np.int64),
                self.col.cpu().numpy().astype(np.int64), v.cpu().numpy())


class HostStreamSpMV:
    """y_host = M x_host for pinned host vectors, the PCIe transfers
    overlapped with the SpMV: x is copied in `chunks` block-row ranges on one
    stream, the SpMV of a row chunk starts as soon as the x chunks holding
    its columns have landed (xdg_bsr_spmv on a row range), and each y chunk
    is copied back on a third stream as soon as it is computed.  Device
    buffers are double-buffered, so back-to-back products overlap too (the
    host <-> device copies run full duplex).  The drop-in analogue of calling
    BlockSparseMatrix.matvec (blockmatrix.py:119-125) on host arrays."""

    def __init__(self, D: "DeviceBSR", chunks: int = 8):
        if D.nbr != D.nbc:
            raise DimensionMismatchError("streamed matvec needs a square operator")
        self.D = D
        dev = D.ctx.device
        rp = D.row_ptr.cpu().numpy().astype(np.int64)
        col = D.col.cpu().numpy().astype(np.int64)
        nbr = D.nbr
        chunks = max(1, min(int(chunks), nbr))
        self.bounds = np.linspace(0, nbr, chunks + 1).round().astype(np.int64)
        # last x chunk each row chunk reads (x chunks land in order)
        rows = np.repeat(np.arange(nbr), np.diff(rp))
        maxcol = np.full(nbr, -1, np.int64)
        np.maximum.at(maxcol, rows, col)
        self.need = []
        for k in range(chunks):
            m = int(maxcol[self.bounds[k]:self.bounds[k + 1]].max(initial=-1))
            self.need.append(max(k, int(np.searchsorted(self.bounds, m, side="right")) - 1))
        n = nbr * D.N
        self.xd = [torch.empty(n, dtype=F64, device=dev) for _ in range(2)]
        self.yd = [torch.empty(n, dtype=F64, device=dev) for _ in range(2)]
        self.s = [torch.cuda.Stream(dev) for _ in range(3)]  # h2d, compute, d2h
        E = torch.cuda.Event
        self.ev_h = [E() for _ in range(chunks)]
        self.ev_c = [E() for _ in range(chunks)]
        self.ev_d = [[E() for _ in range(chunks)] for _ in range(2)]
        self.ev_x = [E() for _ in range(2)]
        self.step = 0

    def launches_per_product(self) -> int:
        return len(self.bounds) - 1

    def __call__(self, xh: torch.Tensor, yh: torch.Tensor, sync: bool = True) -> torch.Tensor:
        """Enqueue one product.  sync=True (default) blocks the host until
        yh holds the product (the reference's matvec returns a finished
        array).  sync=False only enqueues: consecutive products overlap,
        and the caller must call wait() (stream-ordered) and synchronize
        before reading yh on the host."""
        D, N = self.D, self.D.N
        s_h, s_c, s_d = self.s
        buf = self.step & 1
        self.step += 1
        xd, yd = self.xd[buf], self.yd[buf]
        cur = torch.cuda.current_stream(D.ctx.device)
        s_h.wait_stream(cur)
        s_h.wait_event(self.ev_x[buf])  # this x buffer's previous SpMVs are done
        for k in range(len(self.bounds) - 1):
            a, b = int(self.bounds[k]) * N, int(self.bounds[k + 1]) * N
            with torch.cuda.stream(s_h):
                xd[a:b].copy_(xh[a:b], non_blocking=True)
                self.ev_h[k].record(s_h)
        for k in range(len(self.bounds) - 1):
            s_c.wait_event(self.ev_h[self.need[k]])
            s_c.wait_event(self.ev_d[buf][k])  # y chunk of the previous use copied out
            with torch.cuda.stream(s_c):
                D.spmv(xd, yd, rows=(int(self.bounds[k]), int(self.bounds[k + 1])))
                self.ev_c[k].record(s_c)
        self.ev_x[buf].record(s_c)
        for k in range(len(self.bounds) - 1):
            a, b = int(self.bounds[k]) * N, int(self.bounds[k + 1]) * N
            s_d.wait_event(self.ev_c[k])
            with torch.cuda.stream(s_d):
                yh[a:b].copy_(yd[a:b], non_blocking=True)
                self.ev_d[buf][k].record(s_d)
        if sync:
            self.wait()
            s_d.synchronize()  # host-visible: every D2H chunk has landed
        return yh

    def wait(self) -> None:
        """Make the current stream wait for every enqueued copy back.
        Stream-ordered only: it does not block the host."""
        torch.cuda.current_stream(self.D.ctx.device).wait_stream(self.s[2])
