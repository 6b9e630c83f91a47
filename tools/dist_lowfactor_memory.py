"""Per-rank memory of the GMRES-PMG global low-order multifrontal factor
when its elimination subtrees are mapped to P ranks (multifrontal.py:
proportional_map; owned subtrees + replicated top fronts + the received
Schur complements of the cross-rank subtree roots), from the symbolic phase
only (nested dissection + front boundaries, host C++).  Runs this package's
own setup for the BASELINE config (cfg4: 96^3 p=2, k_lo=1 -> 4 low-order
unknowns per block; cfg2: 32^3 p=3, k_lo=2 -> 10), one JSON line per P.

    python tools/dist_lowfactor_memory.py [cfg4|cfg2] [leaf_unknowns]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.case import BenchCase, assemble_case  # noqa: E402
from paper_2003_02431_b200.multifrontal import (SystemGraph, boundaries,  # noqa: E402
                                               nested_dissection, proportional_map)


def main(which="cfg4", leaf=100):
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    if which == "cfg4":
        case = BenchCase(dim=3, cells=96, degree=2, levelset="spheres",
                         levelset_params={"centers": [tuple(-0.4 + c), tuple(0.4 - c)],
                                          "radius": 0.3}, mu_b=100.0, num_levels=4,
                         source="sin", workers=os.cpu_count() or 1)
        m = 4
    else:
        case = BenchCase(dim=3, cells=32, degree=3, levelset="sphere",
                         levelset_params={"center": tuple(c), "radius": 0.6}, mu_a=1.0,
                         mu_b=1000.0, alpha=0.1, num_levels=3, workers=os.cpu_count() or 1)
        m = 10
    t0 = time.perf_counter()
    asm = assemble_case(case)
    lv = asm.hierarchy.level(1)
    rp, col, _ = lv.matrix.bsr_arrays()
    nb = len(rp) - 1
    t1 = time.perf_counter()
    G = SystemGraph(rp, col, [np.arange(nb)])
    P, kids = nested_dissection(G.g_ptr, G.g_col, G.nv, max(1, leaf // m))
    B = boundaries(G.g_ptr, G.g_col, G.nv, P, kids)
    nn = len(P)
    parent = np.full(nn, -1, np.int64)
    for t, ks in enumerate(kids):
        for k in ks:
            parent[k] = t
    pn = np.array([len(x) for x in P], np.float64) * m
    bn = np.array([len(x) for x in B], np.float64) * m
    fb = 8 * (pn * pn + 2 * pn * bn)
    front = 8 * (pn + bn) ** 2
    head = {"case": which, "unknowns": int(nb * m), "fronts": nn, "setup_s": round(t1 - t0, 1),
            "symbolic_s": round(time.perf_counter() - t1, 1),
            "factor_GB_one_gpu": round(fb.sum() / 1e9, 2),
            "largest_front_GB": round(front.max() / 1e9, 2)}
    print(json.dumps(head), flush=True)
    for world in (1, 2, 4, 8):
        r = proportional_map(kids, parent, pn * pn + 2 * pn * bn, world)
        shared = r < 0
        xroot = (r >= 0) & (parent >= 0) & (bn > 0) & (r[np.maximum(parent, 0)] < 0)
        recv = 8 * float((bn[xroot] ** 2).sum())
        per = []
        for q in range(world):
            own = r == q
            per.append((fb[own].sum() + fb[shared].sum()) / 1e9)
        print(json.dumps({"case": which, "ranks": world, "shared_fronts": int(shared.sum()),
                          "replicated_factor_GB": round(fb[shared].sum() / 1e9, 2),
                          "per_rank_factor_GB": [round(v, 2) for v in per],
                          "received_schur_GB": round(recv / 1e9, 2),
                          "largest_shared_front_GB": round(float(front[shared].max()) / 1e9, 2)
                          if shared.any() else 0.0,
                          "max_rank_total_GB": round(max(per) + recv / 1e9 + (
                              float(front[shared].max()) / 1e9 if shared.any() else 0.0), 2)}),
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg4",
         int(sys.argv[2]) if len(sys.argv) > 2 else 100)
