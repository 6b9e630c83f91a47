"""Reference sweep rows for tests/test_bench_api_gpu.py: runs the reference
(cutdg.bench.run_sweep / micro_bench_matops / export_case_matrix) in the
build container and stores its rows (TEST INPUT generation).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_sweep_golden.py
"""
import json
import os
import sys
import tempfile

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from cutdg.bench import (  # noqa: E402
    BenchCase,
    assemble_case,
    export_case_matrix,
    micro_bench_matops,
    run_sweep,
)
from cutdg.solvers import gmres_pmg_solve, ortho_mg_solve  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden import perturbed  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASE = dict(dim=2, cells=8, degree=2, levelset="sphere",
            levelset_params={"center": [0.05, -0.02], "radius": 0.5}, num_levels=2,
            max_iterations=2000, gmres_restart=50, tolerance=1e-8)


def main():
    base = BenchCase(**CASE)
    rows = run_sweep([8], [2], ["direct", "omg", "gmres-pmg"], base_case=base)
    mat = micro_bench_matops(base, repetitions=3)
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "m.mtx")
        n = export_case_matrix(base, p)
        head = open(p).read().splitlines()[:3]
    # +-1-ulp iteration envelopes (SURVEY 8(d) recipe), K = 10 per solver
    asm = assemble_case(base)
    lv = asm.hierarchy.level(1)
    cfg = base.solver_config()
    env = {}
    for solver in ("omg", "gmres-pmg"):
        its = []
        for t in range(10):
            bt = perturbed(lv.rhs, t)
            if solver == "omg":
                _, rep = ortho_mg_solve(asm.hierarchy, bt, None, cfg, 1)
            else:
                _, rep = gmres_pmg_solve(lv.matrix, bt, cfg, dim=base.dim)
            its.append(rep.iterations)
        env[solver] = its
    out = {"case": CASE, "sweep_rows": rows, "matops_rows": mat, "export_dim": n,
           "export_head": head, "envelope": env}
    with open(os.path.join(HERE, "sweep_case.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out)[:800])


if __name__ == "__main__":
    main()
