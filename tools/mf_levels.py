"""Per (level, phase) algorithmic bytes of the multifrontal solve of a
level's low-order system, in launch order -- to pair with an ncu launch
list of the same process (tools/mf_levels_pair.py).  Four-phase plan
(XDG_MF_MERGE=0): gather, lower, bound per level up; upb, upper per level
down.  Merged plan (default): gather, fwd per level up; bwd per level down.

    python tools/mf_levels.py tests/golden/large/cfg2.npz|native [m] [level] > rows.json
"""
import json
import os
import sys

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
ctx = Context.get()
if path == "native":
    from bench import native_cfg2  # noqa: E402

    hier, _, _ = native_cfg2()
    M = hier.level(lam).matrix
    N = M.row_layout.sizes[0]
    nb = M.row_layout.num_blocks
    D = M.device(ctx)
    rp, col = D.row_ptr.cpu().numpy(), D.col.cpu().numpy()
else:
    z = np.load(path)
    rp, col = z[f"L{lam}_row_ptr"], z[f"L{lam}_col"]
    val = fixture_array(z, f"L{lam}_val")
    N = val.shape[1]
    nb = len(rp) - 1
    M = BlockSparseMatrix.from_bsr(rp, col, val, uniform_layout(nb, N), uniform_layout(nb, N))
    D = M.device(ctx)
v = np.arange(nb, dtype=np.int64)
mf = Multifrontal(ctx, rp, col, D.val_t, N, [v], m, v * N, v * m)
pn, bn, h = mf.pn, mf.bn, mf.height
rows = []
for lv in range(mf.nlevels):
    s = h == lv
    ent = int((pn[s] + bn[s]).sum())
    rows.append({"level": lv, "phase": "gather", "bytes": 8 * 4 * ent, "fronts": int(s.sum()),
                 "p_avg": float(pn[s].mean()), "b_avg": float(bn[s].mean())})
    tri, rect = int(4 * (pn[s] ** 2).sum()), int(8 * (pn[s] * bn[s]).sum())
    if mf.merged:
        rows.append({"level": lv, "phase": "fwd", "bytes": tri + rect})
    else:
        rows.append({"level": lv, "phase": "lower", "bytes": tri})
        if rect:
            rows.append({"level": lv, "phase": "bound", "bytes": rect})
for lv in range(mf.nlevels - 1, -1, -1):
    s = h == lv
    tri, rect = int(4 * (pn[s] ** 2).sum()), int(8 * (pn[s] * bn[s]).sum())
    if mf.merged:
        rows.append({"level": lv, "phase": "bwd", "bytes": tri + rect})
    else:
        if rect:
            rows.append({"level": lv, "phase": "upb", "bytes": rect})
        rows.append({"level": lv, "phase": "upper", "bytes": tri})
b = torch.randn(nb * N, dtype=torch.float64, device=ctx.device)
x = torch.zeros(nb * m, dtype=torch.float64, device=ctx.device)
torch.cuda.synchronize()
for _ in range(2):
    mf.solve(b, x)
torch.cuda.synchronize()
print(json.dumps(rows))
