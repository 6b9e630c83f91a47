"""Run-to-run determinism of the native setup and of an OMG solve on it:
hashes of the level operators and right-hand side, then the same solve twice
in this process (iteration counts, solution hashes).  Run it twice to compare
across processes.

    python tools/check_determinism.py [cells] [degree]
"""
import hashlib
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200 import solvers as S  # noqa: E402
from paper_2003_02431_b200.case import BenchCase, assemble_case  # noqa: E402
from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 48
degree = int(sys.argv[2]) if len(sys.argv) > 2 else 3
c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
case = BenchCase(dim=3, cells=cells, degree=degree, levelset="sphere",
                 levelset_params={"center": tuple(c), "radius": 0.5}, mu_b=1000.0, num_levels=3)
A = assemble_case(case)
H = A.hierarchy


def h(a):
    return hashlib.sha1(np.ascontiguousarray(a).tobytes()).hexdigest()[:12]


out = {"levels": []}
for lam in range(1, H.num_levels + 1):
    rp, col, val = H.level(lam).matrix.bsr_arrays()
    out["levels"].append([h(rp), h(col), h(val), h(np.asarray(H.level(lam).rhs))])
lv = H.level(1)
cfg = SolverConfig(tolerance=1e-10, max_iterations=3000, k_lo=(case.resolved_k_lo,),
                   num_levels=3, rm_max_columns=200)
out["solves"] = []
for _ in range(2):
    x, rep = ortho_mg_solve(H, lv.rhs, None, cfg, 1, S._OmgContext(cfg, 1))
    out["solves"].append([rep.iterations, h(np.asarray(x)), h(np.asarray(rep.residual_history))])
print(json.dumps(out))
