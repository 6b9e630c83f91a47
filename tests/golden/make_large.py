"""Serialize a FULL-SIZE reference hierarchy (BASELINE config 2: 3D 32^3,
p=3, sphere r=0.6 with the seed-0 centre, mu 1/1000, f=1, 3 levels) by
running the reference setup (cutdg.bench.assemble_case) in the build
container -- TEST/BENCH INPUT generation, ~15-30 min of CPU.

Writes tests/golden/large/<name>.npz (git-ignored; ~1 GB, travels to the GPU
box with the gpurun snapshot) with the same level arrays as make_golden.py
plus reference outputs that stay cheap at this size: M x at every level,
R x_c / R^T r, and one schwarz_apply at level 1 (k_lo=2, target 2000).

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_large.py cfg2 [cells]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cutdg.bench import BenchCase, assemble_case  # noqa: E402
from cutdg.solvers import schwarz_apply, schwarz_partition  # noqa: E402
from make_golden import bsr_arrays, graph_arrays, ragged  # noqa: E402


def main(name="cfg2", cells=32):
    c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
    case = BenchCase(dim=3, cells=cells, degree=3, levelset="sphere",
                     levelset_params={"center": tuple(c), "radius": 0.6},
                     mu_a=1.0, mu_b=1000.0, alpha=0.1, num_levels=3)
    t0 = time.time()
    asm = assemble_case(case)
    setup = time.time() - t0
    hier = asm.hierarchy
    print(f"[{name}] setup {setup:.0f}s", flush=True)
    out = {}
    rng = np.random.default_rng(20240817)
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        p = f"L{lam}_"
        rp, col, val, N = bsr_arrays(lv.matrix)
        out[p + "row_ptr"], out[p + "col"], out[p + "val"] = rp, col, val
        out[p + "N"] = np.int64(N)
        out[p + "degree"] = np.int64(lv.data.basis.degree)
        out[p + "rhs"] = np.asarray(lv.rhs, float)
        out[p + "adj_ptr"], out[p + "adj"] = graph_arrays(lv.graph)
        x = rng.standard_normal(lv.matrix.shape[1])
        out[p + "x"] = x
        out[p + "Mx"] = lv.matrix.matvec(x)
        if lv.restriction is not None:
            R = lv.restriction
            out[p + "R_row_ptr"], out[p + "R_col"], out[p + "R_val"], _ = bsr_arrays(R)
            out[p + "R_ncols"] = np.int64(R.col_layout.num_blocks)
            xc = rng.standard_normal(R.shape[1])
            out[p + "xc"] = xc
            out[p + "Rxc"] = R.matvec(xc)
            out[p + "Rtr"] = R.transpose().matvec(x)
        print(f"[{name}] level {lam}: {lv.matrix.row_layout.num_blocks} blocks, "
              f"{lv.matrix.num_nonzero_blocks} nnzb", flush=True)
    lv = hier.level(1)
    t0 = time.time()
    part = schwarz_partition(lv.graph, lv.data, max(2000, lv.data.block_size))
    q = "L1_T2000_"
    out[q + "cores_ptr"], out[q + "cores"] = ragged(part.cores)
    out[q + "rows_ptr"], out[q + "rows"] = ragged(part.block_rows)
    out[q + "damping"] = part.damping
    out[q + "schwarz_klo2"] = schwarz_apply(lv.matrix, out["L1_x"], part, 2)
    print(f"[{name}] schwarz k_lo=2 over {part.num_blocks} blocks {time.time() - t0:.0f}s",
          flush=True)
    meta = dict(name=name, dim=3, cells=cells, degree=3, num_levels=hier.num_levels,
                dofs_raw=int(asm.indexmap.L), levelset="sphere",
                levelset_params={"center": list(c), "radius": 0.6},
                setup_seconds=setup,
                omg=dict(tolerance=1e-10, max_iterations=2000, k_lo=2,
                         rm_max_columns=800, num_levels=3),
                gmres=dict(tolerance=1e-10, max_iterations=3000, k_lo=2,
                           gmres_restart=50))
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    os.makedirs(os.path.join(HERE, "large"), exist_ok=True)
    path = os.path.join(HERE, "large", f"{name}.npz")
    np.savez(path, **out)
    print(f"[{name}] wrote {path} ({os.path.getsize(path) / 1e6:.0f} MB)", flush=True)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "cfg2",
         int(sys.argv[2]) if len(sys.argv) > 2 else 32)
