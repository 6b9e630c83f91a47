"""Compare distributed (world=1) OMG pieces against the single-GPU path."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, ".")
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
dist.init_process_group("gloo", rank=0, world_size=1)
from paper_2003_02431_b200 import dist_solvers as DS  # noqa: E402
from paper_2003_02431_b200.blockmatrix import as_block_sparse  # noqa: E402
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.schwarz import schwarz_partition  # noqa: E402
from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve, schwarz_apply  # noqa: E402

z = np.load("tests/golden/bench4.npz")
meta = json.loads(bytes(z["meta"]).decode())
hier = load_hierarchy(z)
ctx = Context.get()
comm = DS.Comm()
for lam in (1, 2):
    lv = hier.level(lam)
    rp, col, val = as_block_sparse(lv.matrix).bsr_arrays()
    N = val.shape[1]
    P = DS.balanced_row_starts(len(rp) - 1, 1)
    part = schwarz_partition(lv.graph, lv.data, max(2000, N))
    S = DS._DistSchwarz(rp, col, val, N, part, min(DS.space_dimension(1, 3), N), P, comm, ctx, None)
    x = np.random.default_rng(0).standard_normal(len(lv.rhs))
    zd = torch.zeros(len(x), dtype=torch.float64, device="cuda")
    S(torch.from_numpy(x).cuda(), zd)
    zs = schwarz_apply(lv.matrix, x, part, 1)
    print("level", lam, "schwarz diff", np.abs(zd.cpu().numpy() - zs).max(), np.abs(zs).max())
    M = DS._DistOp(DS.local_operator(rp, col, val, N, P, 0, ctx), P, comm, ctx, None)
    y = torch.zeros(len(x), dtype=torch.float64, device="cuda")
    M(torch.from_numpy(x).cuda(), y)
    print("level", lam, "spmv diff", np.abs(y.cpu().numpy() - lv.matrix.matvec(x)).max())
    if lv.restriction is not None:
        R = as_block_sparse(lv.restriction)
        Rrp, Rcol, Rval = R.bsr_arrays()
        nc = R.col_layout.num_blocks
        Pc = DS.balanced_row_starts(nc, 1)
        Trp, Tcol, Tval = DS._transpose_bsr(Rrp, Rcol, Rval, nc)
        Rt = DS._DistOp(DS.local_rect_operator(Trp, Tcol, Tval, N, Pc, P, 0, ctx), P, comm, ctx, None)
        yc = torch.zeros(nc * N, dtype=torch.float64, device="cuda")
        Rt(torch.from_numpy(x).cuda(), yc)
        print("level", lam, "Rt diff", np.abs(yc.cpu().numpy() - R.transpose().matvec(x)).max())
cfg = SolverConfig(**meta["omg"])
x1, r1 = ortho_mg_solve(hier, hier.level(1).rhs, None, cfg, 1)
x2, _, r2 = DS.dist_ortho_mg_solve(hier, np.asarray(hier.level(1).rhs), cfg)
print("single", r1.iterations, r1.residual_history[:6])
print("dist  ", r2.iterations, r2.residual_history[:6])
