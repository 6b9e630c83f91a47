"""cProfile the solver setup on a fixture (one OMG iteration)."""
import cProfile
import json
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve  # noqa: E402

path = sys.argv[1]
z = np.load(path)
meta = json.loads(bytes(z["meta"]).decode())
t0 = time.time()
hier = load_hierarchy(z)
print(f"load_hierarchy {time.time() - t0:.2f}s")
lv = hier.level(1)
cfgd = dict(meta["omg"])
cfgd["max_iterations"] = 1
cfg = SolverConfig(**cfgd)
torch.zeros(1).cuda()
pr = cProfile.Profile()
pr.enable()
t0 = time.time()
x, rep = ortho_mg_solve(hier, lv.rhs, None, cfg, 1)
torch.cuda.synchronize()
pr.disable()
print(f"solve(1 it) {time.time() - t0:.2f}s  report {rep.time_iterations:.2f}s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(28)
