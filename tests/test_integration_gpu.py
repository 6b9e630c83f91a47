"""The drop-in boundary exactly as INTEGRATION.md documents it.

* §2: the ctypes stub a maintainer would add to cutdg is extracted from
  INTEGRATION.md and executed verbatim; its matvec must be bit-identical to
  the reference's csr_matvec output (golden fixture) and the C oracle.
* §1: the reference's own setup (`cutdg.bench.assemble_case`, installed
  under baseline/_ref) feeding this package's `solve_assembled`
  (reference bench.py:209-236); skipped when cutdg is not importable.
* the drop-in `BlockSparseMatrix.matvec` on host arrays (pinned staging +
  the overlapped HostStreamSpMV) is bit-identical to the device SpMV.
"""
import os
import re
import sys

import numpy as np
import pytest

from conftest import ROOT, golden_path

pytestmark = pytest.mark.gpu

REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def _snippet(section: str) -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    part = text.split(section, 1)[1]
    m = re.search(r"```python\n(.*?)```", part, re.S)
    return m.group(1)


def _cutdg():
    if REF_SITE not in sys.path and os.path.isdir(REF_SITE):
        sys.path.append(REF_SITE)
    try:
        import cutdg.bench  # noqa: F401
    except Exception as exc:  # noqa: BLE001
        pytest.skip(f"reference cutdg not importable ({exc!r}); "
                    f"install it with tools/install_reference.sh")
    return sys.modules["cutdg.bench"]


def test_integration_ctypes_stub_verbatim():
    from oracle import spmv as ospmv
    from paper_2003_02431_b200 import _native
    from paper_2003_02431_b200.hierarchy import load_hierarchy

    _native.load()  # the in-tree library; the stub's bare CDLL resolves to it (DT_SONAME)
    ns = {}
    exec(compile(_snippet("## 2. C-ABI binding"), "INTEGRATION.md#2", "exec"), ns)
    z = np.load(golden_path("cfg1"))
    hier = load_hierarchy(z)
    for lam in range(1, hier.num_levels + 1):
        M = hier.level(lam).matrix
        M.blocks  # dict-of-blocks form, like the reference's container
        dev = ns["to_device"](M)
        x = z[f"L{lam}_x"]
        y = ns["matvec"](dev, x)
        assert np.array_equal(y, z[f"L{lam}_Mx"]), f"level {lam}: stub != reference matvec"
        rp, col, val = M.bsr_arrays()
        assert np.array_equal(y, ospmv.bsr_spmv(rp, col, val, x))


def test_blockmatrix_matvec_host_arrays_streamed():
    """BlockSparseMatrix.matvec(numpy) goes through pinned staging and the
    overlapped HostStreamSpMV; numpy in -> numpy out, bit-identical; a
    pinned torch tensor in (with out=) is the zero-staging form."""
    import torch

    from oracle import cfg3
    from oracle import spmv as ospmv
    from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout

    rp, col, val, x = cfg3.build(24)
    nb = len(rp) - 1
    lay = uniform_layout(nb, 10)
    M = BlockSparseMatrix.from_bsr(rp, col, val, lay, lay)
    ref = ospmv.bsr_spmv(rp, col, val, x)
    y = M.matvec(x)
    assert isinstance(y, np.ndarray) and np.array_equal(y, ref)
    assert M._host_stream is not None, "host arrays must take the streamed path"
    y2 = M.matvec(x * 2.0)  # buffers reused: the first result must stay intact
    assert np.array_equal(y, ref) and np.array_equal(y2, ospmv.bsr_spmv(rp, col, val, 2 * x))
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(len(x), dtype=torch.float64).pin_memory()
    out = M.matvec(xh, out=yh)
    assert out.data_ptr() == yh.data_ptr() and np.array_equal(yh.numpy(), ref)
    with pytest.raises(Exception):
        M.matvec(x[:-1])


def test_integration_reference_setup_to_b200_solve():
    """INTEGRATION.md §1 with live reference objects: cutdg's setup, this
    package's solve_assembled (GMRES-PMG, OMG, direct) on BASELINE config 1."""
    RB = _cutdg()
    from paper_2003_02431_b200.bench import solve_assembled

    z = np.load(golden_path("cfg1"))
    env = np.load(golden_path("cfg1_env"))
    xd = z["L1_direct_rhs"]
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 2)
    base = dict(dim=2, cells=16, degree=2, levelset="sphere",
                levelset_params={"center": tuple(c), "radius": 0.5}, mu_a=1.0, mu_b=1000.0,
                alpha=0.1, num_levels=3, k_lo=1, tolerance=1e-10)
    asm = RB.assemble_case(RB.BenchCase(**base))
    # the reference's own level-1 system is the one the fixture holds
    lv = asm.hierarchy.level(1)
    assert np.array_equal(np.asarray(lv.rhs), z["L1_rhs"])
    for solver, extra, key in (("gmres-pmg", dict(gmres_restart=50, max_iterations=2000),
                                "gmres_tol1e-10"),
                               ("omg", dict(max_iterations=1000), "omg_tol1e-10"),
                               ("direct", {}, None)):
        case = RB.BenchCase(solver=solver, **base, **extra)
        x, rep = solve_assembled(case, asm)
        assert rep.converged, solver
        assert np.linalg.norm(x - xd) <= 1e-8 * np.linalg.norm(xd), solver
        if key is not None:
            lo, hi = int(env[key].min()), int(env[key].max())
            assert lo - 1 <= rep.iterations <= hi + 1, (solver, rep.iterations, lo, hi)
        assert rep.residual_history[-1] == rep.final_residual
