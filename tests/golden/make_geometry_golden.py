"""Golden cut-cell geometry from the REFERENCE (cutdg.cutcells /
agglomeration) for the setup row SURVEY 8(f)#1: per case the species volumes
of every cell (classify_and_build, cutcells.py:96-197), the small-cell
agglomeration edges (agglomeration.py:41-76) and the level-1 aggregates
(cut_aggregates, agglomeration.py:102-123).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_geometry_golden.py [case ...]
"""
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
from cutdg.agglomeration import (  # noqa: E402
    cut_aggregates,
    lift_aggregation_to_cutcells,
    small_cell_agglomeration_map,
    union_maps,
)
from cutdg.cutcells import classify_and_build  # noqa: E402
from cutdg.levelset import make_level_set  # noqa: E402
from cutdg.mesh import build_cartesian, build_multigrid_aggregation_sequence  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def centre(seed, dim):
    return tuple(np.random.default_rng(seed).uniform(-0.1, 0.1, dim))


CASES = {
    "geo_cfg1": dict(dim=2, cells=16, degree=2, ls="sphere",
                     params=lambda: {"center": centre(0, 2), "radius": 0.5}),
    "geo_bench4": dict(dim=3, cells=4, degree=2, ls="paper-benchmark", params=lambda: {}),
    "geo_sphere8": dict(dim=3, cells=8, degree=3, ls="sphere",
                        params=lambda: {"center": centre(0, 3), "radius": 0.6}),
    "geo_sphere16": dict(dim=3, cells=16, degree=3, ls="sphere",
                         params=lambda: {"center": centre(0, 3), "radius": 0.6}),
    "geo_sphere12_p5": dict(dim=3, cells=12, degree=5, ls="sphere",
                            params=lambda: {"center": centre(0, 3), "radius": 0.5}),
    "geo_cfg2": dict(dim=3, cells=32, degree=3, ls="sphere",
                     params=lambda: {"center": centre(0, 3), "radius": 0.6}),
}


def run(name):
    c = CASES[name]
    alpha = 0.1 if c["degree"] <= 3 else 0.3
    params = c["params"]()
    ls = make_level_set(c["ls"], params)
    mesh = build_cartesian([(-1.0, 1.0)] * c["dim"], [c["cells"]] * c["dim"])
    t0 = time.time()
    cm = classify_and_build(mesh, ls, 3, c["degree"] + 2)
    small = small_cell_agglomeration_map(cm, alpha)
    aggs = cut_aggregates(small)
    edges = np.array(sorted((a[0], a[1], b[0], b[1]) for a, b in small.edges),
                     np.int64).reshape(-1, 4)
    ptr = np.zeros(len(aggs) + 1, np.int64)
    flat = []
    for i, g in enumerate(aggs):
        ptr[i + 1] = ptr[i] + len(g)
        flat += [j * 2 + s for j, s in g]
    # aggregates of hierarchy levels 2..4 (transfer.py:496-500: lifted
    # background axis blocks of width 2^(l-1) united with the small-cell map)
    levels = {}
    for lam, bg in enumerate(build_multigrid_aggregation_sequence(mesh, 4)[1:], start=2):
        eff = union_maps(lift_aggregation_to_cutcells(bg, cm), small)
        g = cut_aggregates(eff)
        lp = np.zeros(len(g) + 1, np.int64)
        lf = []
        for i, grp in enumerate(g):
            lp[i + 1] = lp[i] + len(grp)
            lf += [j * 2 + s for j, s in grp]
        levels[f"L{lam}_agg_ptr"] = lp
        levels[f"L{lam}_agg_pieces"] = np.array(lf, np.int64)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **levels,
                        species_volume=cm.species_volume, small_edges=edges,
                        agg_ptr=ptr, agg_pieces=np.array(flat, np.int64),
                        dim=c["dim"], cells=c["cells"], degree=c["degree"],
                        gauss_order=c["degree"] + 2, quad_depth=3, alpha=alpha,
                        levelset=c["ls"], center=np.array(params.get("center", ())),
                        radius=params.get("radius", 0.0))
    print(f"[{name}] {time.time() - t0:.1f}s cut={len(cm.cut_cells())} aggs={len(aggs)}",
          flush=True)


if __name__ == "__main__":
    for n in sys.argv[1:] or [k for k in CASES if k != "geo_cfg2"]:
        run(n)
