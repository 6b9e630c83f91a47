"""Time the multifrontal solve (xdg_mf_solve) on a fixture's level operator.

    python tools/bench_mf.py tests/golden/large/cfg2.npz [m] [level]
    python tools/bench_mf.py native [m] [level]   # cfg2 from this package's setup

Builds the factor of the level's low-order system (leading m modes of
every block; m = N: the full operator), times solves with CUDA events on the
launching stream and reports algorithmic GB/s (factor + vector bytes)."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout  # noqa: E402
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.hierarchy import fixture_array  # noqa: E402
from paper_2003_02431_b200.multifrontal import Multifrontal  # noqa: E402

path = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
lam = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if path == "native":  # BASELINE cfg2 built by this package's own setup
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from bench import native_cfg2  # noqa: E402

    hier, _, _ = native_cfg2()
    rp = col = None
    M = hier.level(lam).matrix
    N = M.row_layout.sizes[0]
    nb = M.row_layout.num_blocks
else:
    z = np.load(path)
    rp, col = z[f"L{lam}_row_ptr"], z[f"L{lam}_col"]
    val = fixture_array(z, f"L{lam}_val")
    N = val.shape[1]
    nb = len(rp) - 1
    M = BlockSparseMatrix.from_bsr(rp, col, val, uniform_layout(nb, N), uniform_layout(nb, N))
ctx = Context.get()
D = M.device(ctx)
if rp is None or path == "native":
    rp, col = D.row_ptr.cpu().numpy(), D.col.cpu().numpy()
v = np.arange(nb, dtype=np.int64)
b = torch.randn(nb * N, dtype=torch.float64, device=ctx.device)
ref = None
# XDG_MF_FUSE_SWEEP="0,level:6,tree:4": one plan per fused-level mode, each
# checked bit-identical against the first
# XDG_MF_MERGE_SWEEP="0,1": four-phase and merged-phase plans (compared by
# relative difference: the merged factors round differently)
sweep = [(f, mg) for mg in os.environ.get("XDG_MF_MERGE_SWEEP",
                                          os.environ.get("XDG_MF_MERGE", "1")).split(",")
         for f in os.environ.get("XDG_MF_FUSE_SWEEP",
                                 os.environ.get("XDG_MF_FUSE", "0")).split(",")]
for mode, mg in sweep:
    os.environ["XDG_MF_FUSE"] = mode
    os.environ["XDG_MF_MERGE"] = mg
    t0 = time.perf_counter()
    mf = Multifrontal(ctx, rp, col, D.val_t, N, [v], m, v * N, v * m)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    x = torch.zeros(nb * m, dtype=torch.float64, device=ctx.device)
    for _ in range(3):
        mf.solve(b, x)
    ts = []
    for _ in range(20):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        mf.solve(b, x)
        e.record()
        e.synchronize()
        ts.append(s.elapsed_time(e))
    ms = statistics.median(ts)
    # residual of the solve against the level operator's low-order part
    # (torch ops: checker only)
    rpt = torch.from_numpy(np.asarray(rp)).to(ctx.device).long()
    rows_ = torch.repeat_interleave(torch.arange(nb, device=ctx.device), rpt[1:] - rpt[:-1])
    colt = torch.from_numpy(np.asarray(col)).to(ctx.device).long()
    blo = D.val_t.view(-1, N, N)[:, :m, :m].transpose(1, 2)
    ax = torch.zeros(nb, m, dtype=torch.float64, device=ctx.device)
    ax.index_add_(0, rows_, torch.bmm(blo, x.view(nb, m)[colt].unsqueeze(2)).squeeze(2))
    blo_ = b.view(nb, N)[:, :m]
    resid = float((ax - blo_).norm() / blo_.norm())
    if ref is None:
        ref = x.clone()
    # backward error of the solve against the level operator's low-order part
    print(json.dumps({"lib": os.environ.get("XDG_LIB", "default"), "fuse": mode,
                      "merged": bool(mf.merged), "m": m, "rel_residual": resid,
                      "rel_diff_vs_first": float((x - ref).norm() / ref.norm()),
                      "level": lam, "unknowns": nb * m, "nodes": mf.nnodes,
                      "levels": mf.nlevels, "factor_GB": mf.factor_bytes / 1e9,
                      "setup_s": round(setup, 3),
                      "times": {k: round(v, 3) for k, v in mf.times.items()},
                      "solve_ms": ms, "min_ms": min(ts), "GBs": mf.apply_bytes / ms / 1e6,
                      "bit_identical": bool(torch.equal(x, ref))}), flush=True)
    del mf
