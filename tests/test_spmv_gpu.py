"""Device BSR SpMV (xdg_bsr_spmv) parity: bit-exact against the reference's
matvec (golden fixtures) and the C oracle; fused epilogues; full-size
properties at BASELINE config 3 (128^3)."""
import numpy as np
import pytest
import torch

from conftest import golden_path
from oracle import cfg3, spmv as ospmv

pytestmark = pytest.mark.gpu
TOL = 1e-12  # north_star: matvec within 1e-12 relative (we assert bit-exact)


def dev_bsr(rp, col, val, nbc=None):
    from paper_2003_02431_b200.device import DeviceBSR

    N = val.shape[1]
    return DeviceBSR.from_arrays(rp, col, val, N, nbc or (len(rp) - 1))


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3"])
def test_spmv_bitexact_vs_reference_golden(case):
    z = np.load(golden_path(case))
    lam = 1
    while f"L{lam}_row_ptr" in z:
        p = f"L{lam}_"
        D = dev_bsr(z[p + "row_ptr"], z[p + "col"], z[p + "val"])
        y = D.spmv(cuda(z[p + "x"])).cpu().numpy()
        assert np.array_equal(y, z[p + "Mx"]), (case, lam)
        if p + "R_row_ptr" in z:
            R = dev_bsr(z[p + "R_row_ptr"], z[p + "R_col"], z[p + "R_val"],
                        int(z[p + "R_ncols"]))
            assert np.array_equal(R.spmv(cuda(z[p + "xc"])).cpu().numpy(), z[p + "Rxc"])
            # R^T r (the OMG restriction, solvers.py:730): the cached block
            # transpose the solver uses, bit-identical to R.transpose().matvec
            from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout

            N = int(z[p + "N"])
            Rm = BlockSparseMatrix.from_bsr(
                z[p + "R_row_ptr"], z[p + "R_col"], z[p + "R_val"],
                uniform_layout(len(z[p + "R_row_ptr"]) - 1, N),
                uniform_layout(int(z[p + "R_ncols"]), N))
            Rt = Rm.transpose().device()
            assert np.array_equal(Rt.spmv(cuda(z[p + "x"])).cpu().numpy(), z[p + "Rtr"])
        lam += 1


@pytest.mark.parametrize("N", [1, 3, 4, 6, 7, 10, 20, 35, 40, 56])
def test_spmv_block_sizes_vs_oracle(N):
    rng = np.random.default_rng(N)
    nbr = 300
    rows, cols = [], []
    for i in range(nbr):
        nb = rng.integers(0, 9)
        cs = np.unique(np.concatenate([[i], rng.integers(0, nbr, nb)]))
        rows += [i] * len(cs)
        cols += list(cs)
    rp = np.zeros(nbr + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=nbr), out=rp[1:])
    val = rng.standard_normal((len(cols), N, N))
    x = rng.standard_normal(nbr * N)
    D = dev_bsr(rp, np.array(cols), val)
    y = D.spmv(cuda(x)).cpu().numpy()
    assert np.array_equal(y, ospmv.bsr_spmv(rp, cols, val, x))


def test_spmv_empty_rows_and_ranges():
    rng = np.random.default_rng(5)
    N, nbr = 10, 50
    rp = np.zeros(nbr + 1, np.int64)
    rp[1:] = np.cumsum((np.arange(nbr) % 3 == 0).astype(np.int64))
    col = np.flatnonzero(np.arange(nbr) % 3 == 0)
    val = rng.standard_normal((len(col), N, N))
    x = rng.standard_normal(nbr * N)
    D = dev_bsr(rp, col, val)
    ref = ospmv.bsr_spmv(rp, col, val, x)
    y = torch.full((nbr * N,), 7.0, dtype=torch.float64, device="cuda")
    D.spmv(cuda(x), y, rows=(10, 20))
    yh = y.cpu().numpy()
    assert np.array_equal(yh[100:200], ref[100:200])
    assert np.all(yh[:100] == 7.0) and np.all(yh[200:] == 7.0)


def test_spmv_fused_epilogues():
    rp, col, val, x = cfg3.build(8)
    D = dev_bsr(rp, col, val)
    ref = ospmv.bsr_spmv(rp, col, val, x)
    b = np.random.default_rng(3).standard_normal(len(x))
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    r = D.spmv(cuda(x), b=cuda(b), norm_out=nrm).cpu().numpy()
    assert np.array_equal(r, b - ref)
    assert abs(nrm.item() - np.dot(b - ref, b - ref)) <= 1e-12 * np.dot(r, r)
    y0 = cuda(b)
    D.spmv(cuda(x), y0, alpha=2.0, beta=-0.5)
    assert np.allclose(y0.cpu().numpy(), 2.0 * ref - 0.5 * b, rtol=1e-14, atol=1e-12)


def test_spmv_variable_layout_matvec_matches_dense():
    from paper_2003_02431_b200.blockmatrix import BlockLayout, BlockSparseMatrix

    rng = np.random.default_rng(3)
    M = BlockSparseMatrix(BlockLayout((3, 5, 2)), BlockLayout((4, 1, 5)))
    for bi, rs in enumerate((3, 5, 2)):
        for bj, cs in enumerate((4, 1, 5)):
            if rng.uniform() < 0.5 or bi == bj:
                M.add_block(bi, bj, rng.standard_normal((rs, cs)))
    x = rng.standard_normal(10)
    y = M.matvec(x)
    assert np.array_equal(y, M.tocsr() @ x)


def test_spmv_cfg3_32_bitexact_vs_oracle():
    rp, col, val, x = cfg3.build(32)
    D = dev_bsr(rp, col, val)
    y = D.spmv(cuda(x)).cpu().numpy()
    assert np.array_equal(y, ospmv.bsr_spmv(rp, col, val, x, 4))


@pytest.mark.parametrize("chunks", [1, 5, 16])
def test_host_stream_spmv_bitexact(chunks):
    """HostStreamSpMV (host x -> chunked H2D || row-range SpMVs || D2H y,
    double-buffered): bit-identical to the oracle for back-to-back
    products with different inputs, whatever the chunking."""
    from paper_2003_02431_b200.device import HostStreamSpMV

    rp, col, val, x = cfg3.build(24)
    D = dev_bsr(rp, col, val)
    hs = HostStreamSpMV(D, chunks=chunks)
    xs = [np.random.default_rng(k).standard_normal(len(x)) for k in range(3)]
    xh = [torch.from_numpy(v).pin_memory() for v in xs]
    yh = [torch.empty(len(x), dtype=torch.float64).pin_memory() for _ in xs]
    for a, b in zip(xh, yh):
        hs(a, b, sync=False)
    hs.wait()
    torch.cuda.synchronize()
    for v, b in zip(xs, yh):
        assert np.array_equal(b.numpy(), ospmv.bsr_spmv(rp, col, val, v, 4))


@pytest.mark.slow
def test_spmv_cfg3_full_size_properties():
    """128^3 (BASELINE cfg3): rows sampled from the device matrix are
    recomputed by the oracle bit-exactly; linearity holds to roundoff."""
    from paper_2003_02431_b200.synthetic import cfg3_slab_device

    s = cfg3_slab_device(128)
    D = s["D"]
    assert D.nbr == 2202010 and D.nnzb == 14927530
    g = torch.Generator(device="cuda").manual_seed(7)
    L = D.nbr * D.N
    x = torch.randn(L, generator=g, device="cuda", dtype=torch.float64)
    x2 = torch.randn(L, generator=g, device="cuda", dtype=torch.float64)
    y = D.spmv(x)
    # sampled rows against the oracle
    rows = np.sort(np.random.default_rng(0).choice(D.nbr, 2000, replace=False))
    rp = D.row_ptr.cpu().numpy().astype(np.int64)
    ks = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in rows])
    sub_rp = np.concatenate([[0], np.cumsum(rp[rows + 1] - rp[rows])])
    vt = D.val_t[torch.from_numpy(ks).cuda()]
    val = vt.transpose(1, 2).contiguous().cpu().numpy()
    col = D.col.cpu().numpy()[ks].astype(np.int64)
    yref = ospmv.bsr_spmv(sub_rp, col, val, x.cpu().numpy())
    ydev = y.view(-1, D.N)[torch.from_numpy(rows).cuda()].reshape(-1).cpu().numpy()
    assert np.array_equal(ydev, yref)
    # linearity
    lhs = D.spmv(2.0 * x - 3.0 * x2)
    rhs = 2.0 * y - 3.0 * D.spmv(x2)
    rel = (torch.linalg.norm(lhs - rhs) / torch.linalg.norm(rhs)).item()
    assert rel <= TOL
