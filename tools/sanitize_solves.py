"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): SpMV, batched factorization, PMG / Schwarz applies,
rm_step, a few GMRES-PMG (cooperative MGS, ticket-counter reductions) and
OMG (graph-captured: conditional nodes, device-side RM decisions) iterations
on the bench4 / cfg1 hierarchies, plus a multifrontal solve."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch

    from conftest import golden_path
    from paper_2003_02431_b200.device import Context
    from paper_2003_02431_b200.direct import SparseDirect
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.solvers import (SolverConfig, gmres_pmg_solve, ortho_mg_solve,
                                               pmg_apply, schwarz_apply, schwarz_partition)

    ctx = Context.get()
    for case in ("bench4", "cfg1"):
        z = np.load(golden_path(case))
        h = load_hierarchy(z)
        lv = h.level(1)
        x = z["L1_x"]
        dim = 2 if case == "cfg1" else 3
        lv.matrix.matvec(x)
        pmg_apply(lv.matrix, x, 1, range(lv.matrix.row_layout.num_blocks), {}, dim=dim)
        part = schwarz_partition(lv.graph, lv.data, 300)
        schwarz_apply(lv.matrix, x, part, 1)
        gmres_pmg_solve(lv.matrix, lv.rhs, SolverConfig(tolerance=1e-10, max_iterations=60,
                                                        k_lo=1, gmres_restart=50), dim=dim)
        ortho_mg_solve(h, lv.rhs, None, SolverConfig(tolerance=1e-10, max_iterations=8,
                                                     k_lo=1, rm_max_columns=5), 1)
        sd = SparseDirect(lv.matrix.device(ctx), ctx)
        sd.apply(torch.from_numpy(np.asarray(lv.rhs)).to(ctx.device))
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()
