"""Golden data for BASELINE config 5's p-sweep generator at reduced size
("oracle at 12^3-16^3 with the same generator"): sphere r=0.5
with the seed-0 centre, mu 1/1000, f = 1, p = 1..5 with the reference's
default alpha / k_lo (bench.py:56-64), 3-level hierarchy.  Runs the
reference's own assemble_case and solvers (TEST INPUT generation).

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \\
        python tests/golden/make_cfg5_golden.py [cells] [degrees...]
"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cutdg.bench import BenchCase, default_k_lo  # noqa: E402

import make_golden as MG  # noqa: E402


def main(cells=10, degrees=(1, 2, 3, 4, 5)):
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    for p in degrees:
        name = f"cfg5_{cells}_p{p}"
        k_lo = min(default_k_lo(p), p)
        MG.CASES[name] = dict(
            case=BenchCase(dim=3, cells=cells, degree=p, levelset="sphere",
                           levelset_params={"center": tuple(c), "radius": 0.5},
                           mu_a=1.0, mu_b=1000.0, num_levels=3),
            omg=dict(tolerance=1e-8, max_iterations=3000, k_lo=k_lo, num_levels=3),
            gmres=dict(tolerance=1e-8, max_iterations=4000, k_lo=k_lo, gmres_restart=50),
            envelope=5, schwarz_targets=(2000,),
        )
        MG.run(name)


if __name__ == "__main__":
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    degs = tuple(int(a) for a in sys.argv[2:]) or (1, 2, 3, 4, 5)
    main(cells, degs)
