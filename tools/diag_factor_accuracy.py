"""Accuracy of the dense low-order Schwarz solves (diagnostic): forward
error of x = U^-1 L^-1 P b with the triangular inverses from
xdg_batched_factor vs LAPACK LU substitution and vs LAPACK-computed
triangular inverses, against an iteratively refined reference."""
import json
import os
import sys

import numpy as np
import scipy.linalg as sla
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.factor import batched_factor  # noqa: E402


def systems(case, tgt, m):
    z = np.load(os.path.join(ROOT, "tests", "golden", f"{case}.npz"))
    rp, col, val = z["L1_row_ptr"], z["L1_col"], z["L1_val"]
    ptr, rows = z[f"L1_T{tgt}_rows_ptr"], z[f"L1_T{tgt}_rows"]
    out = []
    for s in range(len(ptr) - 1):
        S = rows[ptr[s]:ptr[s + 1]]
        loc = {int(v): i for i, v in enumerate(S)}
        A = np.zeros((len(S) * m,) * 2)
        for i, v in enumerate(S):
            for k in range(rp[v], rp[v + 1]):
                j = loc.get(int(col[k]))
                if j is not None:
                    A[i * m:(i + 1) * m, j * m:(j + 1) * m] = val[k][:m, :m]
        out.append(A)
    return out


def refined(A, b):
    lu = sla.lu_factor(A)
    x = sla.lu_solve(lu, b)
    for _ in range(3):
        r = (b.astype(np.longdouble) - A.astype(np.longdouble) @ x.astype(np.longdouble))
        x = x + sla.lu_solve(lu, r.astype(np.float64))
    return x


def main():
    ctx = Context.get()
    rng = np.random.default_rng(0)
    res = []
    for case, tgt, m in (("cfg1", 300, 6), ("cfg1", 300, 3), ("sphere8p3", 400, 10)):
        if not os.path.exists(os.path.join(ROOT, "tests", "golden", f"{case}.npz")):
            continue
        mats = systems(case, tgt, m)
        flat = np.concatenate([a.ravel() for a in mats])
        off = np.cumsum([0] + [a.size for a in mats[:-1]])
        ns = [a.shape[0] for a in mats]
        A = torch.from_numpy(flat).cuda()
        A2 = A.clone()
        perm, poff, info = batched_factor(ctx, A, off, ns, invert=True)
        F = A.cpu().numpy()
        pm = perm.cpu().numpy()
        batched_factor(ctx, A2, off, ns, invert=False)
        F2 = A2.cpu().numpy()
        e_mine, e_lapack, e_linv, e_myLU_subst, e_myLU_inv, e_lu_diff = [], [], [], [], [], []
        for a, o, po, n in zip(mats, off, poff, ns):
            b = rng.standard_normal(n)
            xr = refined(a, b)
            X = F[o:o + n * n].reshape(n, n)
            pr = pm[po:po + n]
            y = (np.tril(X, -1) + np.eye(n)) @ b[pr]
            x1 = np.triu(X) @ y
            lu, piv = sla.lu_factor(a)
            x2 = sla.lu_solve((lu, piv), b)
            L = np.tril(lu, -1) + np.eye(n)
            U = np.triu(lu)
            Li = sla.solve_triangular(L, np.eye(n), lower=True, unit_diagonal=True)
            Ui = sla.solve_triangular(U, np.eye(n))
            sp = np.arange(n)
            for i, q in enumerate(piv):
                sp[[i, q]] = sp[[q, i]]
            x3 = Ui @ (Li @ b[sp])
            # my LU (no inverse) with LAPACK substitution / LAPACK inverses
            LU2 = F2[o:o + n * n].reshape(n, n)
            L2 = np.tril(LU2, -1) + np.eye(n)
            U2 = np.triu(LU2)
            x4 = sla.solve_triangular(U2, sla.solve_triangular(L2, b[pr], lower=True,
                                                                unit_diagonal=True))
            L2i = sla.solve_triangular(L2, np.eye(n), lower=True, unit_diagonal=True)
            U2i = sla.solve_triangular(U2, np.eye(n))
            x5 = U2i @ (L2i @ b[pr])
            e_lu_diff.append(float(np.abs(LU2 - lu).max() / np.abs(lu).max())
                             if np.array_equal(pr, sp) else -1.0)
            nr = np.linalg.norm(xr)
            e_myLU_subst.append(np.linalg.norm(x4 - xr) / nr)
            e_myLU_inv.append(np.linalg.norm(x5 - xr) / nr)
            e_mine.append(np.linalg.norm(x1 - xr) / nr)
            e_lapack.append(np.linalg.norm(x2 - xr) / nr)
            e_linv.append(np.linalg.norm(x3 - xr) / nr)
        r = {"case": case, "target": tgt, "m": m, "systems": len(mats), "max_n": max(ns),
             "fwd_err_mine_max": max(e_mine), "fwd_err_lapack_subst_max": max(e_lapack),
             "fwd_err_lapack_inverses_max": max(e_linv),
             "fwd_err_myLU_subst_max": max(e_myLU_subst),
             "fwd_err_myLU_lapack_inverses_max": max(e_myLU_inv),
             "lu_diff_vs_lapack_max (-1: other pivots)": max(e_lu_diff),
             "pivots_equal_lapack": int(sum(d >= 0 for d in e_lu_diff)),
             "fwd_err_mine_med": float(np.median(e_mine)),
             "fwd_err_lapack_inverses_med": float(np.median(e_linv))}
        print(json.dumps(r), flush=True)
        res.append(r)


if __name__ == "__main__":
    main()
