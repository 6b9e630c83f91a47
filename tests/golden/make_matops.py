"""The paper's Table-2 instance through the
REFERENCE: 3D 6^3 cells, k=5 (N=56), paper-benchmark surface.  Saves the raw
cut-cell matrix M (bench.py:333) and the initial restriction R0
(hierarchy.to_level1, bench.py:344) as BSR arrays (deduplicated blocks), the
reference's galerkin_restrict(M, None, R0) result (transfer.py:344-351) and
its micro_bench_matops timings (bench.py:326-352), for the block-SpGEMM
parity tests and the matmat row of the benchmark.

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 python tests/golden/make_matops.py [cells] [degree]
"""
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

from cutdg.bench import BenchCase, assemble_case  # noqa: E402
from cutdg.transfer import galerkin_restrict  # noqa: E402
from dedup_fixture import dedup  # noqa: E402


def bsr(M):
    keys = sorted(M.blocks)
    N = M.row_layout.sizes[0]
    rp = np.zeros(M.row_layout.num_blocks + 1, np.int64)
    np.add.at(rp, np.array([k[0] for k in keys]) + 1, 1)
    return (np.cumsum(rp), np.array([k[1] for k in keys], np.int64),
            np.stack([M.blocks[k] for k in keys]) if keys else np.zeros((0, N, N)))


def main(cells=6, degree=5):
    case = BenchCase(dim=3, cells=cells, degree=degree, levelset="paper-benchmark")
    t0 = time.time()
    asm = assemble_case(case)
    print(f"setup {time.time() - t0:.0f}s", flush=True)
    M, R0 = asm.matrix, asm.hierarchy.to_level1
    v = np.ones(M.shape[1])
    M.matvec(v)
    ts = []
    for _ in range(20):
        t = time.perf_counter()
        M.matvec(v)
        ts.append(time.perf_counter() - t)
    t = time.perf_counter()
    Mc, _ = galerkin_restrict(M, None, R0)
    t_mm = time.perf_counter() - t
    out = {}
    for name, A in (("M", M), ("R0", R0), ("Mc", Mc)):
        rp, col, val = bsr(A)
        u, idx = dedup(val)
        out.update({f"{name}_row_ptr": rp, f"{name}_col": col, f"{name}_val__uniq": u,
                    f"{name}_val__idx": idx, f"{name}_ncols": A.col_layout.num_blocks})
    out.update(matvec_ms=1e3 * float(np.median(ts)), matmat_ms=1e3 * t_mm,
               nonzero_rows=int(np.count_nonzero(np.diff(M.tocsr().indptr))),
               cells=cells, degree=degree)
    os.makedirs(os.path.join(HERE, "large"), exist_ok=True)
    path = os.path.join(HERE, "large", f"matops_{cells}_k{degree}.npz")
    np.savez(path, **out)
    print(f"wrote {path} ({os.path.getsize(path) / 1e6:.0f} MB) matvec {out['matvec_ms']:.2f} ms "
          f"matmat {out['matmat_ms']:.1f} ms nnz rows {out['nonzero_rows']}", flush=True)


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
