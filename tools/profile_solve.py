"""Run a solve on a fixture for ncu.

python tools/profile_solve.py <fixture> <omg|gmres> [max_iterations] [--steady]

--steady: warm the solver caches with a first (short) solve, then bracket a
second solve of max_iterations with cudaProfilerStart/Stop, so
`ncu --profile-from-start off` sees only steady-state iteration kernels."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.solvers import (  # noqa: E402
    SolverConfig, _OmgContext, gmres_pmg_solve, ortho_mg_solve)

args = [a for a in sys.argv[1:] if not a.startswith("--")]
steady = "--steady" in sys.argv
path, solver = args[0], args[1]
maxit = int(args[2]) if len(args) > 2 else None
z = np.load(path)
meta = json.loads(bytes(z["meta"]).decode())
hier = load_hierarchy(z)
lv = hier.level(1)
cfgd = dict(meta[solver])
if maxit:
    cfgd["max_iterations"] = maxit
cfg = SolverConfig(**cfgd)
ctx = _OmgContext(cfg, 1)
cache = {}


def run():
    if solver == "omg":
        return ortho_mg_solve(hier, lv.rhs, None, cfg, 1, ctx)
    return gmres_pmg_solve(lv.matrix, lv.rhs, cfg, cache, dim=meta["dim"])


if steady:
    run()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
x, rep = run()
torch.cuda.synchronize()
if steady:
    torch.cuda.profiler.stop()
times = [rep.time_iterations]
for a in sys.argv:  # --repeat=N: N more timed solves in this process
    if a.startswith("--repeat="):
        for _ in range(int(a.split("=")[1])):
            x, rep = run()
            torch.cuda.synchronize()
            times.append(rep.time_iterations)
print(f"{solver}: it={rep.iterations} res={rep.final_residual:.3e} t={rep.time_iterations:.3f}s"
      + (f" all={[round(t, 3) for t in times]}" if len(times) > 1 else ""))
