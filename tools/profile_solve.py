"""Run one solve on a fixture (for ncu launch lists / captures):
python tools/profile_solve.py <fixture path> <omg|gmres> [max_iterations]"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve, ortho_mg_solve  # noqa: E402

path, solver = sys.argv[1], sys.argv[2]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else None
z = np.load(path)
meta = json.loads(bytes(z["meta"]).decode())
hier = load_hierarchy(z)
lv = hier.level(1)
cfgd = dict(meta[solver])
if maxit:
    cfgd["max_iterations"] = maxit
cfg = SolverConfig(**cfgd)
if solver == "omg":
    x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1)
else:
    x, rep = gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=meta["dim"])
torch.cuda.synchronize()
print(f"{solver}: it={rep.iterations} res={rep.final_residual:.3e} t={rep.time_iterations:.3f}s")
