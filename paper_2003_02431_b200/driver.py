"""ctypes mirror of the native solver-driver structs (include/xdg_b200.h,
"Native solver driver") and builders that fill them from the device objects
(DeviceBSR, pmg.PmgPlan, direct.DeviceDirect, RM buffers).

The structs hold plain device pointers; the Python objects owning those
buffers are kept alive by the `_keep` lists of the wrappers below.
"""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as nat

F64 = torch.float64
_vp = C.c_void_p


class XdgBsr(C.Structure):
    _fields_ = [("nbr", C.c_int32), ("nbc", C.c_int32), ("N", C.c_int32),
                ("pad0", C.c_int32), ("nnzb", C.c_int64), ("row_ptr", _vp),
                ("col", _vp), ("val_t", _vp)]


class XdgPmg(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("nsys", "nwork", "N", "m", "has_high",
                                         "direct")] + [("total", C.c_int64)] + \
        [(f, _vp) for f in ("row_sys", "scratch", "lu_off", "dims", "vec_off", "LU",
                            "src", "xlo",
                            "wi_ptr", "wi_blk", "wi_lcol", "wi_cell", "wi_lrow",
                            "wi_xlo", "wi_hidx", "wi_out", "HLU", "hperm", "out",
                            "cptr", "cpos", "damping")] + [("apply_bytes", C.c_double), ("mf", _vp),
                                          ("task_sys", _vp), ("task_row0", _vp),
                                          ("ntasks", C.c_int64),
                                          ("rows_per_task", C.c_int32),
                                          ("max_dim", C.c_int32)]


class XdgDirect(C.Structure):
    _fields_ = [("n", C.c_int32), ("pad0", C.c_int32), ("LU", _vp), ("perm", _vp),
                ("zero_off", _vp), ("dims", _vp), ("row_sys", _vp), ("scratch", _vp),
                ("mf", _vp), ("task_sys", _vp), ("task_row0", _vp), ("ntasks", C.c_int64),
                ("rows_per_task", C.c_int32), ("max_dim", C.c_int32)]


class XdgRm(C.Structure):
    _fields_ = [("n", C.c_int64), ("max_columns", C.c_int32), ("ncols", C.c_int32),
                ("last_dependent", C.c_int32), ("dependent_count", C.c_int32),
                ("rejected_count", C.c_int32), ("restart_count", C.c_int32),
                ("best_norm", C.c_double)] + \
        [(f, _vp) for f in ("W", "Z", "x0", "r0", "y", "My", "My_new", "Mz", "coeff",
                            "sc", "alpha_host", "x", "r", "ws", "gemv_ws")]


class XdgOmgLevel(C.Structure):
    _fields_ = [("M", XdgBsr), ("R", XdgBsr), ("Rt", XdgBsr),
                ("has_restriction", C.c_int32), ("pad0", C.c_int32),
                ("schwarz", XdgPmg), ("direct", XdgDirect), ("rm", XdgRm),
                ("b", _vp), ("z", _vp), ("xf", _vp)]


def _p(t):
    return None if t is None else t.data_ptr()


def bsr_struct(D) -> XdgBsr:
    return XdgBsr(D.nbr, D.nbc, D.N, 0, D.nnzb, D.row_ptr.data_ptr(),
                  D.col.data_ptr(), D.val_t.data_ptr())


def pmg_struct(plan):
    """(XdgPmg, keepalive) for a pmg.PmgPlan."""
    s = XdgPmg()
    s.nsys, s.nwork, s.N, s.m = plan.nsys, plan.nwork, plan.N, plan.m
    s.has_high, s.direct, s.total = int(plan.has_high), int(plan.direct), plan.total
    s.row_sys, s.scratch = _p(plan.row_sys), _p(plan.lu_scratch)
    s.lu_off, s.dims, s.vec_off = _p(plan.lu_off), _p(plan.dims), _p(plan.vec_off)
    s.LU, s.src, s.xlo = _p(plan.LU), _p(plan.src), _p(plan.xlo)
    for f in ("wi_ptr", "wi_blk", "wi_lcol", "wi_cell", "wi_lrow"):
        setattr(s, f, _p(getattr(plan, f)))
    if plan.has_high:
        s.wi_xlo, s.wi_hidx, s.HLU, s.hperm = (_p(plan.wi_xlo), _p(plan.wi_hidx),
                                               _p(plan.HLU), _p(plan.hperm))
    s.wi_out = _p(plan.wi_out) if plan.wi_out is not None else None
    if not plan.direct:
        s.out, s.cptr, s.cpos = _p(plan.out), _p(plan.cptr), _p(plan.cpos)
        s.damping = _p(plan.damping)
    s.apply_bytes = float(plan.algorithmic_bytes())
    if getattr(plan, "task_sys", None) is not None:
        s.task_sys, s.task_row0 = _p(plan.task_sys), _p(plan.task_row0)
        s.ntasks, s.rows_per_task, s.max_dim = (int(plan.task_sys.numel()),
                                                plan.rows_per_task, plan.max_dim)
    keep = []
    if plan.mf is not None:
        ms = plan.mf.struct()
        s.mf = C.addressof(ms)
        keep.append(ms)
    return s, keep


def direct_struct(dd):
    """XdgDirect for a direct.DeviceDirect."""
    s = XdgDirect()
    s.n = dd.n
    if getattr(dd, "mf", None) is not None:
        ms = dd.mf.struct()
        s.mf = C.addressof(ms)
        return s, [ms]
    if dd.n:
        s.LU, s.perm = _p(dd.INV), _p(dd.perm)
        s.zero_off, s.dims = _p(dd.lu_off), _p(dd.dims)
        s.row_sys, s.scratch = _p(dd.row_sys), _p(dd.scratch)
    return s, []


class RmBuffers:
    """Device buffers of one RmState + its XdgRm struct."""

    def __init__(self, ctx, n: int, max_columns: int, allocate_space: bool = True):
        dev = ctx.device
        self.ctx = ctx
        self.n, self.max_columns = n, max_columns
        cols = max_columns if allocate_space else 1
        self.W = torch.empty(cols, n, dtype=F64, device=dev)
        self.Z = torch.empty(cols, n, dtype=F64, device=dev)
        self.vec = torch.zeros(8, n, dtype=F64, device=dev)  # x0 r0 y My My_new Mz x r
        self.coeff = torch.zeros(3 * max(max_columns, 1), dtype=F64, device=dev)
        self.sc = torch.zeros(16, dtype=F64, device=dev)
        self.alpha_host = np.zeros(max(max_columns, 1))
        self.ws = torch.zeros((int(ctx.lib.xdg_reduce_workspace_bytes()) + 7) // 8,
                              dtype=F64, device=dev)
        self.gemv_ws = torch.zeros(
            (int(ctx.lib.xdg_gemv_t_workspace_bytes(max(max_columns, 1))) + 7) // 8,
            dtype=F64, device=dev)
        v = self.vec
        s = XdgRm()
        s.n, s.max_columns = n, max_columns
        s.W, s.Z = self.W.data_ptr(), self.Z.data_ptr()
        s.x0, s.r0, s.y, s.My, s.My_new, s.Mz, s.x, s.r = (v[i].data_ptr() for i in range(8))
        s.coeff, s.sc = self.coeff.data_ptr(), self.sc.data_ptr()
        s.alpha_host = self.alpha_host.ctypes.data
        s.ws, s.gemv_ws = self.ws.data_ptr(), self.gemv_ws.data_ptr()
        self.s = s

    def view(self, addr: int) -> torch.Tensor:
        """The (n,) tensor of vec whose data pointer is addr."""
        for i in range(8):
            if self.vec[i].data_ptr() == addr:
                return self.vec[i]
        raise KeyError(addr)

    @property
    def x(self):
        return self.view(self.s.x)

    @property
    def r(self):
        return self.view(self.s.r)

    @property
    def x0(self):
        return self.view(self.s.x0)

    @property
    def r0(self):
        return self.view(self.s.r0)


def check(status, what):
    nat.check(status, what)
