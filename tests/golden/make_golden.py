"""Generate golden fixtures for the solver hot path by running the REFERENCE
(`cutdg`, imported from /root/reference/pkg/src) in this container.

Test infrastructure only.  Run here (not on the GPU box, which has no
/root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py [case ...]

Each case writes tests/golden/<case>.npz holding
  * the level hierarchy the solvers read (level matrices as BSR arrays with
    row-major N x N blocks, right-hand sides, restriction matrices, aggregate
    adjacency graphs) -- the containers of transfer.py:408-453;
  * the reference's outputs on seeded inputs: BlockSparseMatrix.matvec
    (blockmatrix.py:119-125), R / R^T products (solvers.py:730,734),
    pmg_apply (solvers.py:268-305), schwarz_partition / schwarz_apply
    (solvers.py:384-478), an rm_step sequence (solvers.py:559-625),
    ortho_mg_solve (solvers.py:669-749), gmres_pmg_solve (solvers.py:756-846)
    and the direct solve (blockmatrix.py:203-227);
  * iteration-count envelopes under +-1-ulp perturbations of b
    (recipe in 8(d)).
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from cutdg.bench import BenchCase, assemble_case  # noqa: E402
from cutdg.blockmatrix import direct_factor  # noqa: E402
from cutdg.solvers import (  # noqa: E402
    RmState,
    SolverConfig,
    _OmgContext,
    gmres_pmg_solve,
    ortho_mg_solve,
    pmg_apply,
    rm_step,
    schwarz_apply,
    schwarz_partition,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def bsr_arrays(M):
    """(row_ptr, col, val[nnzb,N,N]) in sorted (bi,bj) order == tocsr order."""
    nbr = M.row_layout.num_blocks
    keys = sorted(M.blocks)
    sizes = set(M.row_layout.sizes) | set(M.col_layout.sizes)
    assert len(sizes) == 1, "uniform layouts only"
    N = sizes.pop()
    row_ptr = np.zeros(nbr + 1, np.int64)
    for bi, _ in keys:
        row_ptr[bi + 1] += 1
    row_ptr = np.cumsum(row_ptr)
    col = np.array([bj for _, bj in keys], np.int64)
    val = np.stack([M.blocks[k] for k in keys]) if keys else np.zeros((0, N, N))
    return row_ptr, col, val, N


def graph_arrays(graph):
    ptr = np.zeros(graph.num_cells + 1, np.int64)
    adj = []
    for c, nbs in enumerate(graph.adjacency):
        ptr[c + 1] = ptr[c] + len(nbs)
        adj.extend(nbs)
    return ptr, np.array(adj, np.int64)


def ragged(seqs):
    ptr = np.zeros(len(seqs) + 1, np.int64)
    flat = []
    for i, s in enumerate(seqs):
        ptr[i + 1] = ptr[i] + len(s)
        flat.extend(s)
    return ptr, np.array(flat, np.int64)


def perturbed(b, t):
    if t == 0:
        return b.copy()
    s = np.random.default_rng(100 + t).choice([-1.0, 1.0], size=len(b))
    return b * (1.0 + 2.2e-16 * s)


CASES = {
    # reference tests' curved-interface benchmark (test_solvers.py:84-98)
    "bench4": dict(
        case=BenchCase(dim=3, cells=4, degree=2, levelset="paper-benchmark",
                       num_levels=3),
        omg=dict(tolerance=1e-10, max_iterations=600, k_lo=1, num_levels=3),
        gmres=dict(tolerance=1e-10, max_iterations=1000, k_lo=1),
        envelope=5, schwarz_targets=(2000, 200),
    ),
    # BASELINE config 1: 2D 16^2 p=2, circle r=0.5, seeded centre, 3 levels
    "cfg1": dict(
        case=None,  # built below (needs the seeded centre)
        omg=dict(tolerance=1e-10, max_iterations=1000, k_lo=1, num_levels=3),
        gmres=dict(tolerance=1e-10, max_iterations=2000, k_lo=1,
                   gmres_restart=50),
        envelope=5, schwarz_targets=(2000, 300),
    ),
    # cfg2 geometry on a smaller grid (p=3, N=20): 8^3, sphere r=0.6
    "sphere8p3": dict(
        case=None,
        omg=dict(tolerance=1e-8, max_iterations=2000, k_lo=2,
                 rm_max_columns=800, num_levels=3),
        gmres=dict(tolerance=1e-8, max_iterations=3000, k_lo=2,
                   gmres_restart=50),
        envelope=5, schwarz_targets=(2000, 400),
    ),
}


def build_case(name):
    spec = CASES[name]
    if name == "cfg1":
        c = np.random.default_rng(0).uniform(-0.1, 0.1, 2)
        return BenchCase(dim=2, cells=16, degree=2, levelset="sphere",
                         levelset_params={"center": tuple(c), "radius": 0.5},
                         mu_a=1.0, mu_b=1000.0, alpha=0.1, num_levels=3,
                         gmres_restart=50)
    if name == "sphere8p3":
        c = np.random.default_rng(0).uniform(-0.1, 0.1, 3)
        return BenchCase(dim=3, cells=8, degree=3, levelset="sphere",
                         levelset_params={"center": tuple(c), "radius": 0.6},
                         mu_a=1.0, mu_b=1000.0, alpha=0.1, num_levels=3)
    return spec["case"]


_SOLVE_CTX = None


def _solve_task(task):
    """One reference solve: t = 0 on b, t > 0 on the +-1-ulp perturbed b."""
    solver, t = task
    hier, M, b, spec, dim = _SOLVE_CTX
    cfg = SolverConfig(**spec[solver])
    bt = b if t == 0 else perturbed(b, t)
    t0 = time.time()
    if solver == "omg":
        x, rep = ortho_mg_solve(hier, bt, None, cfg, 1)
    else:
        x, rep = gmres_pmg_solve(M, bt, cfg, dim=dim)
    dt = time.time() - t0
    print(f"  [{solver} trial {t}] it={rep.iterations} {dt:.1f}s", flush=True)
    if t == 0:
        return (solver, t, rep.iterations, x, np.array(rep.residual_history),
                rep.converged, rep.final_residual, dt)
    return (solver, t, rep.iterations, None, None, rep.converged, rep.final_residual, dt)


def run(name):
    spec = CASES[name]
    case = build_case(name)
    t0 = time.time()
    asm = assemble_case(case)
    hier = asm.hierarchy
    print(f"[{name}] setup {time.time() - t0:.1f}s", flush=True)
    out = {}
    meta = dict(name=name, dim=case.dim, cells=case.cells, degree=case.degree,
                num_levels=hier.num_levels, dofs_raw=int(asm.indexmap.L),
                levelset=case.levelset,
                levelset_params={k: list(v) if isinstance(v, tuple) else v
                                 for k, v in case.levelset_params.items()},
                omg=spec["omg"], gmres=spec["gmres"])
    rng = np.random.default_rng(20240817)
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        p = f"L{lam}_"
        rp, col, val, N = bsr_arrays(lv.matrix)
        out[p + "row_ptr"], out[p + "col"], out[p + "val"] = rp, col, val
        out[p + "N"] = np.int64(N)
        out[p + "degree"] = np.int64(lv.data.basis.degree)
        out[p + "rhs"] = np.asarray(lv.rhs, float)
        gp, ga = graph_arrays(lv.graph)
        out[p + "adj_ptr"], out[p + "adj"] = gp, ga
        # reference SpMV on a seeded vector (blockmatrix.py:119-125)
        x = rng.standard_normal(lv.matrix.shape[1])
        out[p + "x"] = x
        out[p + "Mx"] = lv.matrix.matvec(x)
        if lv.restriction is not None:
            R = lv.restriction
            rr, rc, rv, _ = bsr_arrays(R)
            out[p + "R_row_ptr"], out[p + "R_col"], out[p + "R_val"] = rr, rc, rv
            out[p + "R_ncols"] = np.int64(R.col_layout.num_blocks)
            xc = rng.standard_normal(R.shape[1])
            out[p + "xc"] = xc
            out[p + "Rxc"] = R.matvec(xc)
            out[p + "Rtr"] = R.transpose().matvec(x)
        # Schwarz partitions and applications
        for tgt in spec["schwarz_targets"]:
            target = max(tgt, lv.data.block_size)
            part = schwarz_partition(lv.graph, lv.data, target)
            q = f"{p}T{tgt}_"
            out[q + "cores_ptr"], out[q + "cores"] = ragged(part.cores)
            out[q + "rows_ptr"], out[q + "rows"] = ragged(part.block_rows)
            out[q + "damping"] = part.damping
            for klo in range(0, min(lv.data.basis.degree, 2) + 1):
                try:
                    z = schwarz_apply(lv.matrix, x, part, klo)
                    out[q + f"schwarz_klo{klo}"] = z
                except Exception as exc:  # noqa: BLE001
                    print(f"[{name}] schwarz {q} klo={klo}: {exc!r}")
        # PMG on all cells
        allc = tuple(range(lv.matrix.row_layout.num_blocks))
        for klo in range(0, min(lv.data.basis.degree, 2) + 1):
            try:
                out[p + f"pmg_klo{klo}"] = pmg_apply(
                    lv.matrix, x, klo, allc, {}, dim=case.dim)
            except Exception as exc:  # noqa: BLE001
                print(f"[{name}] pmg L{lam} klo={klo}: {exc!r}")
        # direct solve (coarsest-level semantics, blockmatrix.py:203-227)
        if lv.matrix.shape[0] <= 20000:
            out[p + "direct_rhs"] = direct_factor(lv.matrix).apply(lv.rhs)

    lv = hier.level(1)
    M = lv.matrix
    b = np.asarray(lv.rhs, float)
    # rm_step sequence (solvers.py:559-625), max_columns=3 to hit the cap
    cands = rng.standard_normal((7, len(b)))
    cands[4] = 2.5 * cands[3]  # dependent candidate
    out["rm_cands"] = cands
    state = RmState(np.zeros_like(b), b, 3)
    xs, rs, info = [], [], []
    for z in cands:
        x1, r1, state = rm_step(state, z, M)
        xs.append(x1)
        rs.append(r1)
        info.append([state.ncols, int(state.last_dependent),
                     state.dependent_count, state.rejected_count,
                     state.restart_count])
    out["rm_x"], out["rm_r"] = np.array(xs), np.array(rs)
    out["rm_info"] = np.array(info, np.int64)

    # solves: the reference solve (t = 0) and the envelope's perturbed trials
    # are independent; MG_PAR=N runs them in N forked workers (same code,
    # same single-threaded BLAS: identical results, less wall time)
    global _SOLVE_CTX
    _SOLVE_CTX = (hier, M, b, spec, case.dim)
    tasks = [(solver, t) for solver in ("omg", "gmres") for t in range(spec["envelope"])]
    par = int(os.environ.get("MG_PAR", "1"))
    if par > 1:
        import multiprocessing as mp

        with mp.get_context("fork").Pool(par) as pool:
            results = pool.map(_solve_task, tasks, chunksize=1)
    else:
        results = [_solve_task(tk) for tk in tasks]
    for solver in ("omg", "gmres"):
        res = [r for r in results if r[0] == solver]
        res.sort(key=lambda r: r[1])
        _, _, it0, x, hist, conv, fres, dt = res[0]
        print(f"[{name}] {solver}: it={it0} conv={conv} res={fres:.3e} {dt:.1f}s", flush=True)
        out[f"{solver}_x"] = x
        out[f"{solver}_hist"] = hist
        out[f"{solver}_iters"] = np.int64(it0)
        meta[f"{solver}_seconds"] = dt
        its = [r[2] for r in res]
        out[f"{solver}_envelope"] = np.array(its, np.int64)
        print(f"[{name}] {solver} envelope {its}", flush=True)
    out["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    path = os.path.join(HERE, f"{name}.npz")
    tmp = path + ".tmp.npz"
    np.savez_compressed(tmp, **out)
    if os.path.getsize(tmp) > 8_000_000:  # large fixtures stay out of git
        os.makedirs(os.path.join(HERE, "large"), exist_ok=True)
        path = os.path.join(HERE, "large", f"{name}.npz")
    os.replace(tmp, path)
    print(f"[{name}] wrote {path} ({os.path.getsize(path) / 1e6:.2f} MB)")


if __name__ == "__main__":
    for n in sys.argv[1:] or list(CASES):
        run(n)
