"""ctypes binding of the sm_100a C-ABI (include/xdg_b200.h).

The library is built in-tree by :mod:`._build` (``libxdg_b200.so``).  There
is no CPU fallback: if the library is missing or no CUDA device is present,
every product entry point raises :class:`NativeLibraryError`.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import (
    DimensionMismatchError,
    NativeLibraryError,
    SingularSystemError,
)

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XDG_LIB", os.path.join(_PKG, "libxdg_b200.so"))

XDG_OK, XDG_ERR_ARG, XDG_ERR_CUDA, XDG_ERR_SINGULAR, XDG_ERR_UNSUPPORTED = range(5)

_i32, _i64, _f64, _vp = C.c_int, C.c_int64, C.c_double, C.c_void_p

# name -> (restype, argtypes); must mirror include/xdg_b200.h
SIGNATURES = {
    "xdg_version": (_i32, []),
    "xdg_struct_sizes": (_i32, [_vp, _i32]),
    "xdg_last_error": (C.c_char_p, []),
    "xdg_reduce_workspace_bytes": (_i64, []),
    "xdg_blocks_transpose": (_i32, [_i64, _i32, _vp, _vp, _vp]),
    "xdg_gather_blocks": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp]),
    "xdg_gather_modes": (_i32, [_i64, _i32, _i32, _vp, _vp, _vp]),
    "xdg_bsr_spmv": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp, _f64,
                            _f64, _vp, _vp, _vp, _vp]),
    "xdg_dot": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp]),
    "xdg_axpy": (_i32, [_i64, _f64, _vp, _vp, _vp, _vp]),
    "xdg_scale": (_i32, [_i64, _f64, _vp, _i32, _vp, _vp, _vp]),
    "xdg_sub": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "xdg_add": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "xdg_rm_update": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xdg_div": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "xdg_gemv_t_workspace_bytes": (_i64, [_i32]),
    "xdg_gemv_t": (_i32, [_i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp]),
    "xdg_gemv_update2": (_i32, [_i64, _i32, _vp, _vp, _i64, _vp, _vp, _vp, _vp,
                                _vp]),
    "xdg_add_small": (_i32, [_i32, _vp, _vp, _vp, _vp]),
    "xdg_lu_inv_apply": (_i32, [_i32, _i64] + [_vp] * 10),
    "xdg_lu_inv_apply_tasks": (_i32, [_i64, _vp, _vp, _i32, _i32, _i64] + [_vp] * 9),
    "xdg_ipiv_to_perm": (_i32, [_i32, _vp, _vp, _vp, _vp, _vp]),
    "xdg_pmg_build_low": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp, _vp,
                                 _vp, _vp, _vp, _vp, _vp]),
    "xdg_pack_square": (_i32, [_i64, _vp, _vp, _vp, _i32, _vp, _vp, _i32, _vp]),
    "xdg_pmg_gather_high": (_i32, [_i32, _i32, _i32, _vp, _vp, _vp, _vp,
                                   _vp]),
    "xdg_pmg_high": (_i32, [_i32, _i32, _i32] + [_vp] * 15),
    "xdg_pmg_combine": (_i32, [_i32, _i32, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xdg_galerkin": (_i32, [_i32, _i32] + [_vp] * 8),
    "xdg_assemble_blocks": (_i32, [_i32, _i32] + [_vp] * 9),
    "xdg_rm_step": (_i32, [_vp, _vp, _vp, _vp]),
    "xdg_rm_normalize": (_i32, [_i64, _vp, _vp, _vp, _vp]),
    "xdg_rm_commit": (_i32, [_i64] + [_vp] * 9),
    "xdg_rm_restart_vec": (_i32, [_i64] + [_vp] * 7),
    "xdg_scatter_add_blocks": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp]),
    "xdg_rm_init": (_i32, [_vp, _vp, _vp, _vp]),
    "xdg_rm_restart": (_i32, [_vp, _vp]),
    "xdg_rm_current": (_i32, [_vp, _vp]),
    "xdg_pmg_apply_op": (_i32, [_vp, _vp, _vp, _vp, _vp]),
    "xdg_omg_solve": (_i32, [_vp, _i32, _i32, _f64, _i32, _i32, _vp, _vp, _i32,
                             _vp, _vp, _vp, _vp, _vp, _vp]),
    "xdg_gmres_solve": (_i32, [_vp, _vp, _i32, _f64, _i32, _vp, _vp, _i32]
                        + [_vp] * 14),
    "xdg_mgs": (_i32, [_i64, _i32, _vp, _i64, _vp, _vp, _vp, _vp]),
    "xdg_mf_solve": (_i32, [_vp, _vp, _vp, _vp]),
    "xdg_nd_order": (_i64, [_i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "xdg_nd_boundaries": (_i64, [_i64, _vp, _vp, _i64, _vp, _vp, _vp]),
    "xdg_nd_boundaries_copy": (_i32, [_vp, _vp]),
    "xdg_schwarz_partition": (_i64, [_i64, _vp, _vp, _vp, _i64]),
    "xdg_schwarz_sizes": (_i32, [_vp]),
    "xdg_schwarz_copy": (_i32, [_vp, _vp, _vp, _vp]),
    "xdg_mf_rows_per_warp": (_i32, []),
    "xdg_mf_merge": (_i32, [_i64, _i32, _i32, _vp, _vp, _vp, _vp]),
    "xdg_mf_extend_add": (_i32, [_i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "xdg_batched_factor": (_i32, [_i64, _vp, _vp, _vp, _vp, _i32, _i32, _vp, _vp, _vp,
                                  _vp, _i32, _vp, _vp]),
    "xdg_batched_factor_ws_bytes": (_i64, [_i64, _i32]),
    "xdg_axpy_dot": (_i32, [_i64, _f64, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "xdg_mf_solve_phase": (_i32, [_vp, _vp, _vp, _i32, _vp]),
    "xdg_scatter_blocks": (_i32, [_i64, _i32, _vp, _vp, _vp, _vp]),
}

_lib = None
_lock = threading.Lock()


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeLibraryError(
                f"{path} not built: run `python -c 'import __graft_entry__ as g;"
                f" g.build()'` (there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().xdg_last_error().decode(errors="replace")


def check(status: int, what: str = "") -> None:
    if status == XDG_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if status == XDG_ERR_ARG:
        raise DimensionMismatchError(msg)
    if status == XDG_ERR_SINGULAR:
        raise SingularSystemError(msg)
    raise NativeLibraryError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
