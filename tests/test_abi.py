"""The C-ABI library loads and exports every symbol include/xdg_b200.h
declares (no GPU needed: nothing is computed)."""
import ctypes
import os
import re

from conftest import ROOT

from paper_2003_02431_b200 import _build, _native


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "xdg_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(xdg_\w+)\(",
                                 text, flags=re.M)))


def test_header_declares_the_hot_path():
    syms = declared_symbols()
    for need in ("xdg_bsr_spmv", "xdg_dot", "xdg_gemv_t", "xdg_gemv_update2",
                 "xdg_lu_inv_apply", "xdg_pmg_high",
                 "xdg_rm_step", "xdg_omg_solve", "xdg_gmres_solve", "xdg_mgs", "xdg_pmg_combine",
                 "xdg_rm_update", "xdg_blocks_transpose"):
        assert need in syms


def test_library_builds_and_exports_every_declared_symbol():
    lib_path = _build.build()
    lib = ctypes.CDLL(lib_path)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    # and the Python binding covers exactly the header
    assert sorted(_native.SIGNATURES) == declared_symbols()


def test_binding_loads_without_gpu():
    lib = _native.load()
    assert lib.xdg_version() >= 1
    assert lib.xdg_reduce_workspace_bytes() > 0


def test_ctypes_struct_layouts_match_the_header():
    """The ctypes mirrors of the driver structs have the C sizes (a field
    added on one side only would shift every pointer after it)."""
    import ctypes as C

    import numpy as np

    from paper_2003_02431_b200 import _native as nat
    from paper_2003_02431_b200.driver import XdgBsr, XdgDirect, XdgOmgLevel, XdgPmg, XdgRm
    from paper_2003_02431_b200.multifrontal import NODE_DT, XdgMf

    out = np.zeros(16, np.int64)
    k = nat.load().xdg_struct_sizes(out.ctypes.data, 16)
    assert k == 7
    mine = [C.sizeof(XdgBsr), C.sizeof(XdgPmg), C.sizeof(XdgDirect), C.sizeof(XdgRm),
            C.sizeof(XdgOmgLevel), C.sizeof(XdgMf), NODE_DT.itemsize]
    assert list(out[:k]) == mine
