"""cProfile of the lazy solver setup (inside the solve timer, like the
reference) on a fixture hierarchy: OMG context (Schwarz partitions, PMG
plans, coarse factor, transposes) and the GMRES-PMG plan.

    python tools/profile_setup_solve.py tests/golden/large/cfg2.npz [omg|gmres]
"""
import cProfile
import json
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.hierarchy import load_hierarchy  # noqa: E402
from paper_2003_02431_b200.solvers import (  # noqa: E402
    SolverConfig, _OmgContext, gmres_pmg_solve, ortho_mg_solve)

path, solver = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "omg")
if path == "cfg4-native":  # BASELINE config 4 at full size via the native setup
    from paper_2003_02431_b200.case import BenchCase, assemble_case

    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    case = BenchCase(dim=3, cells=int(os.environ.get("CELLS", "96")), degree=2,
                     levelset="spheres",
                     levelset_params={"centers": [tuple(-0.4 + c), tuple(0.4 - c)],
                                      "radius": 0.3}, mu_b=100.0, num_levels=4,
                     source="sin", workers=os.cpu_count() or 1)
    t0 = time.perf_counter()
    hier = assemble_case(case).hierarchy
    print(f"native setup {time.perf_counter() - t0:.1f} s", flush=True)
    meta = {"dim": 3, "omg": {"tolerance": 1e-10, "max_iterations": 1, "k_lo": 1,
                              "num_levels": 4}}
else:
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    hier = load_hierarchy(z)
lv = hier.level(1)
cfgd = dict(meta[solver])
cfgd["max_iterations"] = 1
cfg = SolverConfig(**cfgd)
# warm-up (module loads, cuSOLVER/MAGMA handles) on a tiny system
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.factor import warmup  # noqa: E402
warmup(Context.get())
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
if solver == "omg":
    ortho_mg_solve(hier, lv.rhs, None, cfg, 1, _OmgContext(cfg, 1))
else:
    gmres_pmg_solve(lv.matrix, lv.rhs, cfg, dim=meta["dim"])
torch.cuda.synchronize()
pr.disable()
print(f"{solver} setup + 1 iteration: {time.perf_counter() - t0:.2f} s")
pstats.Stats(pr).sort_stats(os.environ.get("PROFILE_SORT", "cumulative")).print_stats(
    int(os.environ.get("PROFILE_LINES", "35")))
