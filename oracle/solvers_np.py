"""numpy/scipy restatement of the reference solver algorithms -- TEST
INFRASTRUCTURE (checker and timed CPU baseline; never the product path).

Operates on plain arrays: a level is (row_ptr, col, val[nnzb, N, N]
row-major, N); the hierarchy is a list of dicts with the level matrix, its
restriction R (BSR arrays, or None), the aggregate adjacency lists and the
basis degree.  Each function cites the reference lines it restates
(/root/reference/pkg/src/cutdg/solvers.py).  Pinned against the reference's
own outputs in tests/test_oracle.py (golden fixtures).
"""
from __future__ import annotations

from collections import deque
from math import comb
from time import perf_counter

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import scipy.sparse.linalg as spla

DEPENDENT_RTOL = 1e-13  # solvers.py:52


def csr_of(rp, col, val, ncols_blocks=None):
    """CSR of a uniform BSR (== BlockSparseMatrix.tocsr(), blockmatrix.py:91-114)."""
    N = val.shape[1]
    nbr = len(rp) - 1
    nbc = ncols_blocks if ncols_blocks is not None else nbr
    return sp.bsr_matrix((val, np.asarray(col), np.asarray(rp)),
                         shape=(nbr * N, nbc * N)).tocsr()


# ---- degree-separated preconditioner (solvers.py:183-305) -----------------

class PmgFactors:
    """Factors of one (cell set, low-mode count) pair (solvers.py:191-243)."""

    def __init__(self, rp, col, val, cells, m):
        N = val.shape[1]
        cells = np.asarray(cells, np.int64)
        self.cells, self.m, self.N = cells, m, N
        nb = len(rp) - 1
        loc = np.full(nb, -1, np.int64)
        loc[cells] = np.arange(len(cells))
        sub_rows, sub_cols, sub_k = [], [], []
        for i, c in enumerate(cells):
            ks = np.arange(rp[c], rp[c + 1])
            lc = loc[col[ks]]
            keep = lc >= 0
            sub_rows.append(np.full(keep.sum(), i))
            sub_cols.append(lc[keep])
            sub_k.append(ks[keep])
        r = np.concatenate(sub_rows)
        cc = np.concatenate(sub_cols)
        kk = np.concatenate(sub_k)
        srp = np.zeros(len(cells) + 1, np.int64)
        np.cumsum(np.bincount(r, minlength=len(cells)), out=srp[1:])
        self.sub = csr_of(srp, cc, val[kk])                       # solvers.py:208
        self.gidx = (cells[:, None] * N + np.arange(N)).ravel()
        self.low = (np.arange(len(cells))[:, None] * N + np.arange(m)).ravel()
        low = csr_of(srp, cc, np.ascontiguousarray(val[kk][:, :m, :m])).tocsc()
        with np.errstate(all="ignore"):
            self.lu = spla.splu(low)                              # blockmatrix.py:213
        self.high = []
        if m < N:                                                 # solvers.py:225-243
            for i, c in enumerate(cells):
                kd = rp[c] + np.searchsorted(col[rp[c]:rp[c + 1]], c)
                H = np.array(val[kd][m:, m:])
                self.high.append((i * N + np.arange(m, N), sla.lu_factor(H, check_finite=False)))

    def apply(self, b):                                           # solvers.py:245-265
        bl = b[self.gidx]
        xl = np.zeros_like(bl)
        xl[self.low] = self.lu.solve(bl[self.low])
        if self.high:
            r = bl - self.sub @ xl
            for idx, f in self.high:
                xl[idx] += sla.lu_solve(f, r[idx], check_finite=False)
        x = np.zeros_like(b)
        x[self.gidx] = xl
        return x


def modes_low(k_lo, dim, N):
    return min(comb(k_lo + dim, dim), N)                          # solvers.py:288


# ---- Schwarz (solvers.py:384-478) -------------------------------------------

def schwarz_blocks(adjacency, block_size, target):
    """Greedy BFS cores + one-layer extension + damping (solvers.py:384-457),
    for aggregation levels (one block per node)."""
    n = len(adjacency)
    nbrs = [sorted(a) for a in adjacency]
    done = np.zeros(n, bool)
    cores = []
    for seed in range(n):
        if done[seed]:
            continue
        core, got, q, seen = [], 0, deque([seed]), {seed}
        while q and got < target:
            c = q.popleft()
            if done[c]:
                continue
            done[c] = True
            core.append(c)
            got += block_size
            for v in nbrs[c]:
                if not done[v] and v not in seen:
                    seen.add(v)
                    q.append(v)
        cores.append(sorted(core))
    ext = [sorted(set(c).union(*[nbrs[v] for v in c])) for c in cores]
    damping = np.zeros(n * block_size)
    for e in ext:
        for c in e:
            damping[c * block_size:(c + 1) * block_size] += 1.0
    return ext, damping


def schwarz_apply(factors, damping, r):
    z = np.zeros_like(r)
    for F in factors:
        z += F.apply(r)
    return z / damping


# ---- residual minimisation (solvers.py:485-625) ----------------------------

class Rm:
    def __init__(self, x0, r0, cap):
        n = len(x0)
        self.x0, self.r0, self.cap = x0.copy(), r0.copy(), cap
        self.W = np.zeros((n, cap))
        self.Z = np.zeros((n, cap))
        self.y = np.zeros(n)
        self.My = np.zeros(n)
        self.best = float(np.linalg.norm(r0))
        self.k = 0
        self.flags = [0, 0, 0, 0]  # dependent, dependent_count, rejected, restarts

    def current(self):
        return self.x0 + self.y, self.r0 - self.My

    def restart(self):
        self.x0 = self.x0 + self.y
        self.r0 = self.r0 - self.My
        self.y = np.zeros_like(self.y)
        self.My = np.zeros_like(self.My)
        self.best = float(np.linalg.norm(self.r0))
        self.k = 0
        self.flags[3] += 1

    def step(self, z, M):
        if self.k >= self.cap:
            self.restart()
        z = np.array(z, float)
        w = M @ z
        scale = float(np.linalg.norm(w))
        W, Z = self.W[:, :self.k], self.Z[:, :self.k]
        for _ in range(2):
            c = W.T @ w
            w -= W @ c
            z -= Z @ c
        nw = float(np.linalg.norm(w))
        if scale == 0.0 or nw <= DEPENDENT_RTOL * scale:
            self.flags[0] = 1
            self.flags[1] += 1
            return self.current()
        w /= nw
        z /= nw
        a = float(w @ self.r0)
        y_new = self.y + a * z
        My_new = self.My + a * (M @ z)
        rho = float(np.linalg.norm(self.r0 - My_new))
        self.flags[0] = 0
        if rho > self.best:
            self.flags[2] += 1
            self.restart()
            return self.current()
        self.W[:, self.k], self.Z[:, self.k] = w, z
        self.y, self.My, self.best = y_new, My_new, rho
        self.k += 1
        return self.current()


# ---- solvers (solvers.py:669-846) -------------------------------------------

class Hierarchy:
    """levels[i] = dict(M=csr, N, degree, adjacency, R=csr|None, Rt=csr|None,
    rp/col/val BSR arrays) for i = 0 .. L-1 (level 1 first)."""

    def __init__(self, levels, dim):
        self.levels, self.dim = levels, dim
        self.cache = {}

    def smoother(self, lam, target, k_lo):
        key = ("sw", lam, k_lo)
        if key not in self.cache:
            lv = self.levels[lam - 1]
            ext, damp = schwarz_blocks(lv["adjacency"], lv["N"], max(target, lv["N"]))
            m = modes_low(k_lo, self.dim, lv["N"])
            self.cache[key] = ([PmgFactors(lv["rp"], lv["col"], lv["val"], e, m)
                                for e in ext], damp)
        return self.cache[key]

    def direct(self, lam):
        key = ("lu", lam)
        if key not in self.cache:
            with np.errstate(all="ignore"):
                self.cache[key] = spla.splu(self.levels[lam - 1]["M"].tocsc())
        return self.cache[key]


def omg(h: Hierarchy, b, cfg, lam=1, entry=1):
    """Alg. 4 recursion (solvers.py:669-749); returns (x, iterations, history)."""
    lv = h.levels[lam - 1]
    M = lv["M"]
    if lam == len(h.levels) or lv["R"] is None:
        x = h.direct(lam).solve(b)
        res = float(np.linalg.norm(b - M @ x))
        return x, 0, [res]
    x = np.zeros_like(b)
    r = b - M @ x
    st = Rm(x, r, cfg["rm_max_columns"])
    hist = [float(np.linalg.norm(r))]
    facs, damp = h.smoother(lam, cfg["schwarz_target_dofs"], cfg["k_lo"])
    budget = cfg["max_iterations"] if lam == entry else cfg["coarse_cycle_iterations"]
    it = 0
    while hist[-1] > cfg["tolerance"] and it < budget:
        it += 1
        x, r = st.step(schwarz_apply(facs, damp, r), M)
        xc, _, _ = omg(h, lv["Rt"] @ r, cfg, lam + 1, entry)
        x, r = st.step(lv["R"] @ xc, M)
        x, r = st.step(schwarz_apply(facs, damp, r), M)
        hist.append(float(np.linalg.norm(r)))
    return x, it, hist


def gmres(M, rp, col, val, b, cfg, dim, timing=None):
    """Restarted right-preconditioned GMRES with MGS (solvers.py:756-846).
    timing (optional dict): receives "setup_s" (the lazy PMG factorization,
    which the reference counts inside its solve timer, solvers.py:778) and
    "iter_s" (seconds of every iteration) -- for the CPU-baseline tools."""
    import time as _time

    N = val.shape[1]
    _t0 = _time.perf_counter()
    F = PmgFactors(rp, col, val, np.arange(len(rp) - 1), modes_low(cfg["k_lo"], dim, N))
    if timing is not None:
        timing["setup_s"] = _time.perf_counter() - _t0
        timing["iter_s"] = []
    m, tol, maxit = cfg["gmres_restart"], cfg["tolerance"], cfg["max_iterations"]
    x = np.zeros_like(b)
    r = b - M @ x
    beta = float(np.linalg.norm(r))
    hist, total = [beta], 0
    while beta > tol and total < maxit:
        n = len(b)
        V, Z = np.zeros((n, m + 1)), np.zeros((n, m))
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        V[:, 0] = r / beta
        j = 0
        while j < m and total < maxit:
            total += 1
            _ti = _time.perf_counter()
            Z[:, j] = F.apply(V[:, j])
            w = M @ Z[:, j]
            for i in range(j + 1):
                H[i, j] = float(V[:, i] @ w)
                w -= H[i, j] * V[:, i]
            H[j + 1, j] = float(np.linalg.norm(w))
            if H[j + 1, j] > 0.0:
                V[:, j + 1] = w / H[j + 1, j]
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            d = float(np.hypot(H[j, j], H[j + 1, j]))
            cs[j], sn[j] = H[j, j] / d, H[j + 1, j] / d
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            H[j + 1, j] = 0.0
            est = abs(float(g[j + 1]))
            hist.append(est)
            if timing is not None:
                timing["iter_s"].append(_time.perf_counter() - _ti)
            j += 1
            if est <= tol:
                break
        yv = sla.solve_triangular(H[:j, :j], g[:j], check_finite=False)
        x = x + Z[:, :j] @ yv
        r = b - M @ x
        beta = float(np.linalg.norm(r))
        hist[-1] = beta
    return x, total, hist


def hierarchy_from_npz(z, dim):
    """Build the oracle hierarchy from a golden fixture."""
    levels = []
    lam = 1
    while f"L{lam}_row_ptr" in z:
        p = f"L{lam}_"
        rp, col, val = z[p + "row_ptr"], z[p + "col"], z[p + "val"]
        N = int(z[p + "N"])
        ptr, adj = z[p + "adj_ptr"], z[p + "adj"]
        lv = dict(rp=rp, col=col, val=val, N=N, M=csr_of(rp, col, val),
                  degree=int(z[p + "degree"]),
                  adjacency=[list(adj[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)],
                  R=None, Rt=None)
        if p + "R_row_ptr" in z:
            R = csr_of(z[p + "R_row_ptr"], z[p + "R_col"], z[p + "R_val"], int(z[p + "R_ncols"]))
            lv["R"], lv["Rt"] = R, R.T.tocsr()
        levels.append(lv)
        lam += 1
    return Hierarchy(levels, dim)


def timed_solve(z, meta, solver):
    """(x, iterations, seconds) of one oracle solve on a fixture, the timer
    covering the lazy factorisations like the reference (solvers.py:696,778)."""
    h = hierarchy_from_npz(z, meta["dim"])
    cfg = dict(tolerance=1e-10, max_iterations=1000, k_lo=1, schwarz_target_dofs=2000,
               gmres_restart=30, rm_max_columns=200, coarse_cycle_iterations=2)
    cfg.update(meta[solver])
    cfg["k_lo"] = int(cfg["k_lo"][0] if isinstance(cfg["k_lo"], (list, tuple)) else cfg["k_lo"])
    b = np.asarray(z["L1_rhs"], float)
    t0 = perf_counter()
    if solver == "omg":
        x, it, _ = omg(h, b, cfg)
    else:
        lv = h.levels[0]
        x, it, _ = gmres(lv["M"], lv["rp"], lv["col"], lv["val"], b, cfg, meta["dim"])
    return x, it, perf_counter() - t0
