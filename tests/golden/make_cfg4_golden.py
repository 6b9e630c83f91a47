"""Golden data for BASELINE config 4's generator at reduced size (SURVEY
8(d): "oracle at 24^3 with the same generator"; here 8^3 so the reference
finishes in minutes): union of two seeded spheres r=0.3, mu 1:100,
f = sin(pi x) sin(pi y) sin(pi z), Dirichlet, 4-level hierarchy.

The reference has no built-in union level set or sin source (BenchCase
knows "sphere" and f = 1); SURVEY 8(d) prescribes `LevelSet(lambda X:
min(phi1, phi2), grad of the active sphere)` (levelset.py:19-35) and
`dirichlet_problem(1, 100, f, 3)` (assembly.py:89-103).  This script
substitutes exactly those into the reference's own assemble_case
(bench.py:165-206) and runs it here (TEST INPUT generation).

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \\
        python tests/golden/make_cfg4_golden.py [cells]
"""
import os
import sys

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import cutdg.bench as RB  # noqa: E402
from cutdg.levelset import LevelSet, make_level_set  # noqa: E402

import make_golden as MG  # noqa: E402


def centres(seed=0):
    """The two non-overlapping centres of the config-4 generator
    (bench.py CFG4 recipe of this repo): -0.4 + c and 0.4 - c, c seeded."""
    c = np.random.default_rng(seed).uniform(-0.1, 0.1, 3)
    return tuple(-0.4 + c), tuple(0.4 - c)


def union_level_set(params):
    s1 = make_level_set("sphere", {"center": params["centers"][0], "radius": params["radius"]})
    s2 = make_level_set("sphere", {"center": params["centers"][1], "radius": params["radius"]})

    def phi(X):
        return np.minimum(s1(X), s2(X))

    def grad(X):
        first = s1(X) <= s2(X)
        return np.where(first[:, None], s1.gradient(X), s2.gradient(X))

    return LevelSet(phi, grad)


def sin_source(X):
    return np.sin(np.pi * X[:, 0]) * np.sin(np.pi * X[:, 1]) * np.sin(np.pi * X[:, 2])


_make, _dirichlet = RB.make_level_set, RB.dirichlet_problem
RB.make_level_set = lambda name, params=None: (
    union_level_set(params) if name == "spheres" else _make(name, params))
RB.dirichlet_problem = lambda mu_a, mu_b, source, dim, *a, **k: _dirichlet(
    mu_a, mu_b, sin_source, dim, *a, **k)
MG.assemble_case = RB.assemble_case


def main(cells=8):
    c1, c2 = centres()
    name = f"cfg4_{cells}"
    MG.CASES[name] = dict(
        case=RB.BenchCase(dim=3, cells=cells, degree=2, levelset="spheres",
                          levelset_params={"centers": (c1, c2), "radius": 0.3},
                          mu_a=1.0, mu_b=100.0, alpha=0.1, num_levels=4),
        omg=dict(tolerance=1e-8, max_iterations=2000, k_lo=1, num_levels=4),
        gmres=dict(tolerance=1e-8, max_iterations=3000, k_lo=1, gmres_restart=50),
        envelope=5, schwarz_targets=(2000,),
    )
    MG.run(name)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 8)
