"""Multifrontal sparse LU on the device: the stored factorization behind the
large low-order PMG systems, the Schwarz blocks' low-order systems and large
direct / coarsest-level solves.

The reference factors these systems with SuperLU (`splu`, COLAMD + partial
pivoting: cutdg blockmatrix.py:203-227, used by solvers.py:208-221 low-order
PMG factor, 249-251 its solve, 661-666 / 698-710 coarsest level).  Dense
device LU (direct.py) streams 8 n^2 bytes per solve and cannot hold the
global low-order system of a 32^3 p=3 case at all (336,610 unknowns ->
906 GB).  Here:

* symbolic (host, setup): the block graph of every system is ordered by
  nested dissection (BFS level-set separators from a pseudo-peripheral
  vertex, recursively), giving an elimination forest of fronts.  Front t
  eliminates its pivot blocks P_t against its boundary B_t (the ancestor
  separator blocks adjacent to t's subtree);
* numeric (device, setup; batched cuSOLVER/MAGMA getrf, cuBLAS trsm/GEMM as
  plumbing): fronts of one height are assembled (original blocks + the
  children's Schur complements, child by child -- deterministic), padded
  into size buckets, LU-factored with partial pivoting inside P_t, and
  L_BP = F_BP U^-1, U_PB = L^-1 P F_PB, S = F_BB - L_BP U_PB formed.  The
  triangular factors of every front are stored as explicit inverses (as in
  direct.py), so a solve is only GEMVs;
* solve (xdg_mf_solve, csrc/xdg_multifrontal.cu): 5 row-parallel launches per
  tree height, every system of the forest at once, no atomics.

Pivoting is partial within each front's pivot block (the standard
multifrontal restriction).  The systems are SIP-DG operators (symmetric in
pattern, values symmetric to ~1e-11 relative, positive definite: SURVEY
8(c)), for which this is stable; any exactly zero / non-finite pivot raises
SingularSystemError like SuperLU's "exactly singular" (blockmatrix.py:211-215).
"""
from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np
import torch

from . import _native as nat
from .factor import batched_factor
from .errors import SingularSystemError

F64 = torch.float64
I32 = torch.int32
I64 = torch.int64

NODE_DT = np.dtype([("p", "<i4"), ("b", "<i4"), ("ldp", "<i4"), ("ldb", "<i4"),
                    ("gp", "<i4"), ("gb", "<i4"), ("ldr", "<i4"), ("pad1", "<i4"),
                    ("inv", "<i8"), ("lbp", "<i8"), ("upb", "<i8"), ("w", "<i8"),
                    ("y", "<i8"), ("c", "<i8"), ("bx", "<i8"), ("px", "<i8")])
assert NODE_DT.itemsize == 96
MF_U = 8  # loads in flight per lane per chunk (MF_U, xdg_multifrontal.cu)


def _row_sets() -> int:
    """Row sets per warp task of a short-row front (G < 32 lanes per row):
    2 issues both sets' loads together (bit-identical sums).  XDG_MF_SETS."""
    import os

    v = int(os.environ.get("XDG_MF_SETS", "2"))
    if v not in (1, 2):
        raise ValueError(f"XDG_MF_SETS={v}: expected 1 or 2")
    return v


def _fuse_mode() -> tuple[str, int]:
    """Low levels run as fused launches (xdg_mf.fuse_levels), XDG_MF_FUSE:
    "tree:K" -- one launch per sweep, one CTA per subtree of fronts of
    height < K; "level:K" -- one launch per height < K, one CTA per front
    (gather + lower + bound, upb + upper); "0" -- per-phase launches."""
    import os

    v = os.environ.get("XDG_MF_FUSE", "0")
    if v == "0":
        return "off", 0
    mode, _, k = v.partition(":")
    if mode not in ("tree", "level") or not k.isdigit():
        raise ValueError(f"XDG_MF_FUSE={v}: expected tree:K, level:K or 0")
    return mode, int(k)


def _merge_mode() -> bool:
    """Merged phases (default): the factors hold M = L_BP L^-1 and N = U^-1
    U_PB (xdg_mf_merge), one row launch per height and sweep instead of two.
    XDG_MF_MERGE=0 keeps the four-phase solve (lower, bound, upb, upper);
    the fused low levels (XDG_MF_FUSE) exist for the four-phase solve only."""
    import os

    v = os.environ.get("XDG_MF_MERGE", "1")
    if v not in ("0", "1"):
        raise ValueError(f"XDG_MF_MERGE={v}: expected 0 or 1")
    return v == "1" and _fuse_mode()[0] == "off"


def _long_row() -> int:
    """Merged phases: rows of at least this many elements are CTA tasks (the
    CTA's warps share the row's chunks).  XDG_MF_LONG, default 2048 = one
    chunk of 32 lanes x 8 loads for each of the 8 warps."""
    import os

    return max(1, int(os.environ.get("XDG_MF_LONG", "2048")))


def _col_pivots() -> int:
    """Merged phases: fronts with at most this many (padded) pivot unknowns
    run their forward rows one THREAD per row over a column-major copy of
    [L^-1; M_BP] (coalesced across rows, no reductions or masks: the row-major
    lane groups spend ~2 instructions per matrix entry on fronts of 10-300
    pivots).  XDG_MF_PCOL; 0 (default) disables: measured SLOWER on the cfg2
    low-order system (PCOL 0 / 128 / 320 / 640 -> 2.54 / 2.72 / 2.96 / 3.23 ms,
    profiles/r2_mf_pcol_sweep.jsonl) -- the low levels are bound by the
    dependent loads per task, not by the lane mapping."""
    import os

    return max(0, int(os.environ.get("XDG_MF_PCOL", "0")))


def _rows_per_warp() -> int:
    """Rows a warp task of a whole-warp front covers: the kernel's kMR."""
    return int(nat.load().xdg_mf_rows_per_warp())


_vp = C.c_void_p


class XdgMf(C.Structure):
    _fields_ = [("nlevels", C.c_int32), ("nnodes", C.c_int32), ("total", C.c_int64)] + \
        [(f, _vp) for f in ("lev_ent", "lev_task", "ent_w", "ent_src", "ent_cptr",
                            "ent_cidx", "tasks", "nodes", "bidx",
                            "pdst", "ent_scale", "pscale", "F", "W", "Y", "C")] + \
        [("apply_bytes", C.c_double), ("fuse_levels", C.c_int32), ("nfbatch", C.c_int32),
         ("nfstages", C.c_int64)] + \
        [(f, _vp) for f in ("fb_grp", "g_stage", "st_ent", "st_task", "fent", "ftask")] + \
        [("X", _vp), ("merged", C.c_int32), ("pad_", C.c_int32)]


def _ranges(starts: np.ndarray, ends: np.ndarray) -> np.ndarray:
    lens = ends - starts
    tot = int(lens.sum())
    if tot == 0:
        return np.zeros(0, np.int64)
    offs = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens)
    return np.arange(tot, dtype=np.int64) + offs


# ---------------------------------------------------------------------------
# Systems -> one combined vertex graph

class SystemGraph:
    """Vertices = (system, block) pairs of every system (systems are
    independent components).  `a_*`: the restricted BSR entries (with the
    diagonal) as (row vertex, col vertex, global block index); `g_*`: the
    symmetrised adjacency without self loops (ordering graph)."""

    def __init__(self, rp: np.ndarray, col: np.ndarray, sets):
        rp = np.asarray(rp, np.int64)
        col = np.asarray(col, np.int64)
        nbr = len(rp) - 1
        loc = np.full(nbr, -1, np.int64)
        rows_l, cols_l, ks_l = [], [], []
        base = 0
        gblk, sys_of = [], []
        for s, S in enumerate(sets):
            S = np.asarray(S, np.int64)
            loc[S] = np.arange(len(S)) + base
            ks = _ranges(rp[S], rp[S + 1])
            lc = loc[col[ks]]
            keep = lc >= 0
            rows = np.repeat(np.arange(len(S)) + base, rp[S + 1] - rp[S])
            rows_l.append(rows[keep])
            cols_l.append(lc[keep])
            ks_l.append(ks[keep])
            loc[S] = -1
            gblk.append(S)
            sys_of.append(np.full(len(S), s, np.int64))
            base += len(S)
        cat = (lambda xs: np.concatenate(xs) if xs else np.zeros(0, np.int64))
        self.nv = base
        self.gblk, self.sys = cat(gblk), cat(sys_of)
        self.a_row, self.a_col, self.a_k = cat(rows_l), cat(cols_l), cat(ks_l)
        off = self.a_row != self.a_col
        nv1 = max(self.nv, 1)

        def sorted_unique(k):
            if len(k) > 1 and not np.all(k[1:] > k[:-1]):
                k = np.sort(k)
                k = k[np.concatenate([[True], k[1:] != k[:-1]])]
            return k

        # entries come row by row with ascending columns (sorted BSR rows and
        # sorted sets), so the forward keys are already sorted; a structurally
        # symmetric pattern (every operator here) needs no merge with its
        # transpose.  (np.unique over both copies: 4.6 s of hashing for the
        # 1.6 M vertices of cfg4's Schwarz systems.)
        kf = sorted_unique(self.a_row[off] * nv1 + self.a_col[off])
        kt = sorted_unique(self.a_col[off] * nv1 + self.a_row[off])
        key = kf if (len(kf) == len(kt) and np.array_equal(kf, kt)) else \
            sorted_unique(np.concatenate([kf, kt]))
        r, c = key // nv1, key % nv1
        self.g_ptr = np.zeros(self.nv + 1, np.int64)
        np.cumsum(np.bincount(r, minlength=self.nv), out=self.g_ptr[1:])
        self.g_col = c


# ---------------------------------------------------------------------------
# Nested dissection

class _ND:
    def __init__(self, g_ptr, g_col, nv, leaf):
        self.ptr, self.col, self.leaf = g_ptr, g_col, max(1, int(leaf))
        self.active = np.zeros(nv, bool)
        self.dist = np.full(nv, -1, np.int64)
        self.P = []
        self.kids = []

    def _bfs(self, start):
        dist, ptr, col, act = self.dist, self.ptr, self.col, self.active
        front = np.array([start], np.int64)
        dist[start] = 0
        levels = [front]
        d = 0
        while True:
            nb = col[_ranges(ptr[front], ptr[front + 1])]
            nb = nb[act[nb]]
            nb = np.unique(nb[dist[nb] < 0])
            if nb.size == 0:
                break
            d += 1
            dist[nb] = d
            levels.append(nb)
            front = nb
        for lv in levels:
            dist[lv] = -1
        return levels

    def _node(self, P, kids):
        self.P.append(np.sort(P))
        self.kids.append(kids)
        return len(self.P) - 1

    def run(self, V) -> list:
        V = np.asarray(V, np.int64)
        if V.size == 0:
            return []
        self.active[V] = True
        levels = self._bfs(int(V[0]))
        reached = np.concatenate(levels)
        if reached.size < V.size:
            self.active[V] = False
            rest = np.setdiff1d(V, reached, assume_unique=True)
            return self.run(np.sort(reached)) + self.run(rest)
        if V.size <= self.leaf or len(levels) < 3:
            self.active[V] = False
            return [self._node(V, [])]
        levels = self._bfs(int(levels[-1][0]))
        self.active[V] = False
        if len(levels) < 3:
            return [self._node(V, [])]
        sizes = np.array([len(lv) for lv in levels])
        cum = np.cumsum(sizes)
        n = V.size
        ks = np.arange(1, len(levels) - 1)
        left, right = cum[ks - 1], n - cum[ks]
        k = int(ks[np.argmin(np.maximum(left, right) * 2 + sizes[ks])])
        # thinned separator: the smaller one-sided cut between levels k, k+1
        nxt = np.zeros(len(self.dist), bool)
        nxt[levels[k + 1]] = True
        a1 = self._adjacent(levels[k], nxt)
        cur = np.zeros(len(self.dist), bool)
        cur[levels[k]] = True
        a2 = self._adjacent(levels[k + 1], cur)
        if a2.sum() < a1.sum():
            S = levels[k + 1][a2]
            L = np.concatenate(levels[:k + 1])
            R = np.concatenate([levels[k + 1][~a2]] + levels[k + 2:])
        else:
            S = levels[k][a1]
            L = np.concatenate(levels[:k] + [levels[k][~a1]])
            R = np.concatenate(levels[k + 1:])
        kids = self.run(np.sort(L)) + self.run(np.sort(R))
        return [self._node(S, kids)]

    def _adjacent(self, verts, mark):
        """per vertex of verts: has a neighbour with mark set"""
        if verts.size == 0:
            return np.zeros(0, bool)
        cnt = self.ptr[verts + 1] - self.ptr[verts]
        hit = mark[self.col[_ranges(self.ptr[verts], self.ptr[verts + 1])]]
        owner = np.repeat(np.arange(len(verts)), cnt)
        return np.bincount(owner, weights=hit, minlength=len(verts)) > 0


class _Ragged(list):
    """List of index arrays that are slices of one flat array (`flat`,
    `ptr`): the fronts / boundary sets as the native ordering returns them.
    `_flat` gives the concatenation back without touching the slices."""
    flat = None
    ptr = None


class _Kids(list):
    """Children lists of the fronts with the parent array they were built
    from (`_parent_of` returns it without walking the lists)."""
    parent = None


def _flat(L):
    """(concatenation, lengths) of a list of index arrays."""
    if isinstance(L, _Ragged) and L.flat is not None:
        return L.flat, np.diff(L.ptr)
    n = len(L)
    lens = np.fromiter((len(a) for a in L), np.int64, n)
    return (np.concatenate(L) if n else np.zeros(0, np.int64)), lens


def _parent_of(kids) -> np.ndarray:
    """parent[c] of every front from the children lists (-1: root)."""
    nn = len(kids)
    if isinstance(kids, _Kids) and kids.parent is not None:
        return kids.parent
    parent = np.full(nn, -1, np.int64)
    klen = np.fromiter((len(k) for k in kids), np.int64, nn)
    if klen.sum():
        kcat = np.fromiter((c for k in kids for c in k), np.int64, int(klen.sum()))
        parent[kcat] = np.repeat(np.arange(nn), klen)
    return parent


def nested_dissection(g_ptr, g_col, nv, leaf):
    """Post-ordered elimination forest (P list, children list): the native
    xdg_nd_order (csrc/xdg_ordering.cu); nested_dissection_py is the same
    algorithm in numpy (kept as its test oracle)."""
    g_ptr = np.ascontiguousarray(g_ptr, np.int64)
    g_col = np.ascontiguousarray(g_col, np.int64)
    node_ptr = np.zeros(nv + 1, np.int64)
    verts = np.zeros(max(nv, 1), np.int64)
    parent = np.zeros(max(nv, 1), np.int64)
    nn = int(nat.load().xdg_nd_order(int(nv), g_ptr.ctypes.data, g_col.ctypes.data,
                                      int(leaf), node_ptr.ctypes.data, verts.ctypes.data,
                                      parent.ctypes.data))
    P = _Ragged(verts[node_ptr[t]:node_ptr[t + 1]] for t in range(nn))
    P.flat, P.ptr = verts[:node_ptr[nn]], node_ptr[:nn + 1]
    kids = _Kids([] for _ in range(nn))
    par = parent[:nn]
    for c in np.flatnonzero(par >= 0).tolist():
        kids[par[c]].append(c)
    kids.parent = par.copy()
    return P, kids


def boundaries(g_ptr, g_col, nv, P, kids):
    """B_t of every front (xdg_nd_boundaries): neighbours of t's subtree in
    ancestor fronts, sorted by (owner, vertex)."""
    nn = len(P)
    g_ptr = np.ascontiguousarray(g_ptr, np.int64)
    g_col = np.ascontiguousarray(g_col, np.int64)
    pcat, plen = _flat(P)
    node_ptr = np.zeros(nn + 1, np.int64)
    np.cumsum(plen, out=node_ptr[1:])
    verts = np.ascontiguousarray(pcat, np.int64)
    parent = np.full(max(nn, 1), -1, np.int64)
    parent[:nn] = _parent_of(kids)
    lib = nat.load()
    tot = int(lib.xdg_nd_boundaries(int(nv), g_ptr.ctypes.data, g_col.ctypes.data, nn,
                                    node_ptr.ctypes.data, verts.ctypes.data,
                                    parent.ctypes.data))
    b_ptr = np.zeros(nn + 1, np.int64)
    b_verts = np.zeros(max(tot, 1), np.int64)
    lib.xdg_nd_boundaries_copy(b_ptr.ctypes.data, b_verts.ctypes.data)
    B = _Ragged(b_verts[b_ptr[t]:b_ptr[t + 1]] for t in range(nn))
    B.flat, B.ptr = b_verts[:b_ptr[nn]], b_ptr
    return B


def boundaries_py(g_ptr, g_col, P, kids, owner):
    """numpy restatement of xdg_nd_boundaries (test oracle)."""
    B_list = []
    for t in range(len(P)):
        cand = [g_col[_ranges(g_ptr[P[t]], g_ptr[P[t] + 1])]]
        cand += [B_list[c] for c in kids[t]]
        cand = np.unique(np.concatenate(cand))
        Bt = cand[owner[cand] > t]
        B_list.append(Bt[np.lexsort((Bt, owner[Bt]))])
    return B_list


def nested_dissection_py(g_ptr, g_col, nv, leaf):
    """numpy restatement of xdg_nd_order (test oracle)."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import connected_components

    nd = _ND(g_ptr, g_col, nv, leaf)
    old = sys.getrecursionlimit()
    sys.setrecursionlimit(max(old, 100000))
    try:
        if nv:
            A = csr_matrix((np.ones(len(g_col)), g_col, g_ptr), shape=(nv, nv))
            ncomp, lab = connected_components(A, directed=False)
            order = np.argsort(lab, kind="stable")
            cptr = np.zeros(ncomp + 1, np.int64)
            np.cumsum(np.bincount(lab, minlength=ncomp), out=cptr[1:])
            for c in range(ncomp):
                nd.run(np.sort(order[cptr[c]:cptr[c + 1]]))
    finally:
        sys.setrecursionlimit(old)
    return nd.P, nd.kids


def proportional_map(kids, parent, work, world: int, slack: float = 1.1) -> np.ndarray:
    """Subtree-to-rank mapping of an elimination forest (post-ordered: a
    subtree is the contiguous id range ending at its root) for `world`
    ranks: rank_of[t] = the rank owning front t with its whole subtree, or
    -1 for a shared top front (factored and solved redundantly on every
    rank).  The candidate subtrees start as the forest's roots; while the
    heaviest candidate (subtree factor bytes) exceeds `slack` x the average
    share of a rank, it becomes shared and its children replace it; the
    candidates then go to the least-loaded rank, heaviest first (LPT).
    Deterministic: every rank computes the same map."""
    nn = len(parent)
    rank_of = np.full(nn, -1, np.int64)
    if nn == 0:
        return rank_of
    sub = np.asarray(work, np.float64).copy()
    size = np.ones(nn, np.int64)
    for t in range(nn):
        if parent[t] >= 0:
            sub[parent[t]] += sub[t]
            size[parent[t]] += size[t]
    cand = [t for t in range(nn) if parent[t] < 0]
    while True:
        tot = sum(sub[t] for t in cand)
        h = max(cand, key=lambda t: (sub[t], t))
        if world == 1 or not kids[h] or sub[h] <= slack * tot / world:
            break
        cand.remove(h)
        cand += list(kids[h])
    load = np.zeros(world)
    for t in sorted(cand, key=lambda t: (-sub[t], t)):
        r = int(np.argmin(load))
        load[r] += sub[t]
        rank_of[t - size[t] + 1:t + 1] = r
    # a shared front all of whose subtrees landed on one rank is owned by it
    below = {}
    for t in range(nn):  # post-order: children first
        if rank_of[t] < 0:
            rs = set()
            for c in kids[t]:
                rs |= below[c] if rank_of[c] < 0 else {int(rank_of[c])}
            if len(rs) == 1:
                rank_of[t] = rs.pop()
            below[t] = rs if rank_of[t] < 0 else set()
    return rank_of


def _group(n: int) -> int:
    """Lanes per row for rows of length n: the smallest power of two with
    8 loads per lane covering the row, at most a warp."""
    g = 1
    while g < 32 and MF_U * g < n:
        g *= 2
    return g


def _group_v(n: np.ndarray) -> np.ndarray:
    """_group over an array."""
    g = np.ones(len(n), np.int64)
    for _ in range(5):
        g = np.where((g < 32) & (MF_U * g < n), g * 2, g)
    return g


def _pad(x: int) -> int:
    return x if x <= 32 else ((x + 31) // 32) * 32


# ---------------------------------------------------------------------------

class Multifrontal:
    """Factor of a batch of independent block systems.

    rp, col: BSR pattern (host) of the operator whose blocks are taken;
    val_t: device tensor (nnzb, N, N) of column-major blocks (DeviceBSR.val_t);
    sets: list of sorted block-row arrays (one system each); m: unknowns per
    block (the leading m x m corner of every block is used);
    vsrc / vdst: per combined vertex, index of its mode 0 in the solve's
    input b / output x (mode a adds a)."""

    def __init__(self, ctx, rp, col, val_t, N, sets, m, vsrc, vdst,
                 leaf_unknowns: int = 100, what: str = "system",
                 equilibrate: bool = True, front_factor=None, comm=None):
        import time

        t0 = time.perf_counter()
        self.ctx = ctx
        dev = ctx.device if ctx is not None else val_t.device
        self.m = m = int(m)
        G = SystemGraph(rp, col, sets)
        self.G = G
        nv = G.nv
        self.total = nv * m
        # leaf size of the dissection (unknowns): XDG_MF_LEAF for every plan,
        # XDG_MF_LEAF_MULTI for plans of several independent systems (Schwarz
        # blocks: shallow trees, launch-bound levels)
        leaf_env = os.environ.get("XDG_MF_LEAF_MULTI" if len(sets) > 1 else "XDG_MF_LEAF")
        if leaf_env:
            leaf_unknowns = int(leaf_env)
        P_list, kids = nested_dissection(G.g_ptr, G.g_col, nv, max(1, leaf_unknowns // m))
        nn = len(P_list)
        self.nnodes = nn
        Pcat0, Plen0 = _flat(P_list)
        owner = np.empty(nv, np.int64)
        owner[Pcat0] = np.repeat(np.arange(nn), Plen0)
        parent = np.full(nn, -1, np.int64)
        height = np.zeros(nn, np.int64)
        if nn:
            parent = np.array(_parent_of(kids), np.int64)
            klen = np.bincount(parent[parent >= 0], minlength=nn)
            # post-order ids (children < parent): heights level by level
            lev = np.flatnonzero(klen == 0)
            while len(lev):
                par = parent[lev]
                ok = par >= 0
                np.maximum.at(height, par[ok], height[lev[ok]] + 1)
                lev = np.unique(par[ok])
        # boundaries (post-order: subtree of t has ids < t, ancestors > t)
        B_list = boundaries(G.g_ptr, G.g_col, nv, P_list, kids)
        Bcat0, Blen0 = _flat(B_list)
        pn = Plen0 * m
        bn = Blen0 * m
        self.P_list, self.B_list, self.kids, self.parent = P_list, B_list, kids, parent
        self.height = height
        H = int(height.max()) + 1 if nn else 0
        self.nlevels = H
        pp = np.where(pn <= 32, pn, (pn + 31) // 32 * 32)  # _pad
        bp = np.where(bn <= 32, bn, (bn + 31) // 32 * 32)
        # multi-GPU (comm with world > 1): subtree-to-rank proportional
        # mapping; a rank factors and solves its owned subtrees plus the
        # shared top fronts (replicated), see proportional_map
        self.comm = comm if (comm is not None and comm.world > 1) else None
        self.merged = merged = _merge_mode()
        if self.comm is not None:
            work = (pn * pn + 2 * pn * bn).astype(np.float64)
            self.rank_of = proportional_map(kids, parent, work, self.comm.world)
            me = self.comm.rank
            need = (self.rank_of == me) | (self.rank_of < 0)
        else:
            self.rank_of = np.zeros(nn, np.int64)
            need = np.ones(nn, bool)
        self.need = need
        # roots of owned subtrees whose parent is a shared front: their Schur
        # complements / contributions cross ranks (sorted by (rank, id))
        xroot = np.flatnonzero((self.rank_of >= 0) & (parent >= 0) & (bn > 0)
                               & (self.rank_of[np.maximum(parent, 0)] < 0))
        xroot = xroot[np.lexsort((xroot, self.rank_of[xroot]))] if len(xroot) else xroot
        self.xroot = xroot

        # position of every vertex inside its owner's P; B positions by key
        ppos = np.empty(nv, np.int64)
        ppos[Pcat0] = _ranges(np.zeros(nn, np.int64), Plen0)
        bkey_node = np.repeat(np.arange(nn), Blen0)
        bkey_v = Bcat0
        bkey = bkey_node * max(nv, 1) + bkey_v
        bkey_pos = _ranges(np.zeros(nn, np.int64), Blen0) if nn else bkey
        so = np.argsort(bkey, kind="stable")
        bkey, bkey_pos = bkey[so], bkey_pos[so]

        def bpos(node, v):
            i = np.searchsorted(bkey, node * max(nv, 1) + v)
            return bkey_pos[i]

        def front_pos(node, v):
            """Padded front row of mode 0 of vertex v in node's front."""
            inP = owner[v] == node
            out = np.empty(len(v), np.int64)
            out[inP] = ppos[v[inP]] * m
            nb_ = ~inP
            out[nb_] = pp[node[nb_]] + bpos(node[nb_], v[nb_]) * m
            return out

        t1 = time.perf_counter()
        # ---- factor storage / workspace layout ---------------------------
        order = np.lexsort((np.arange(nn), height))  # by height, then id
        buckets = {}  # (h, pp, bp) -> node list: fronts of the first pass
        buckets_sh = {}  # the shared (replicated) top fronts: second pass
        shared = self.rank_of < 0
        for sel_, bk_ in ((need & ~shared, buckets), (need & shared, buckets_sh)):
            ts_all = order[sel_[order]]
            if not len(ts_all):
                continue
            K = int(max(pp.max(), bp.max())) + 1
            keys = (height[ts_all] * K + pp[ts_all]) * K + bp[ts_all]
            _, first, inv = np.unique(keys, return_index=True, return_inverse=True)
            rank = np.empty(len(first), np.int64)  # buckets in order of first appearance
            rank[np.argsort(first, kind="stable")] = np.arange(len(first))
            so_ = np.argsort(rank[inv], kind="stable")
            cuts = np.flatnonzero(np.diff(rank[inv][so_])) + 1
            for grp in np.split(ts_all[so_], cuts):
                t0_ = int(grp[0])
                bk_[(int(height[t0_]), int(pp[t0_]), int(bp[t0_]))] = grp.tolist()
        inv_off = np.zeros(nn, np.int64)
        lbp_off = np.zeros(nn, np.int64)
        upb_off = np.zeros(nn, np.int64)
        fst = 0
        PCOL = _col_pivots() if merged else 0
        colf = np.zeros(nn, bool)      # forward rows thread-per-row (column-major copy)
        ldr = np.zeros(nn, np.int64)   # its leading dimension (rows, padded to 4)
        for (h, P_, B_), ts in list(buckets.items()) + list(buckets_sh.items()):
            nb = len(ts)
            inv_off[ts] = fst + np.arange(nb) * P_ * P_
            fst += nb * P_ * P_
            if 0 < P_ <= PCOL:
                colf[ts] = True
                ldr[ts] = (P_ + B_ + 3) // 4 * 4
                lbp_off[ts] = fst + np.arange(nb) * P_ * ldr[ts[0]]
                fst += nb * P_ * int(ldr[ts[0]])
                upb_off[ts] = fst + np.arange(nb) * P_ * B_
                fst += nb * P_ * B_
                continue
            lbp_off[ts] = fst + np.arange(nb) * B_ * P_
            fst += nb * B_ * P_
            upb_off[ts] = fst + np.arange(nb) * P_ * B_
            fst += nb * P_ * B_
        # the padded factors plus the largest height's front buffer must fit
        front_max = max((sum(len(ts) * (P_ + B_) ** 2 for bk in (buckets, buckets_sh)
                             for (hh, P_, B_), ts in bk.items() if hh == h)
                         for h in range(H)), default=0)
        # received Schur complements of the cross-rank subtree roots
        xs_sz = int(sum(int(bn[t]) ** 2 for t in self.xroot))
        free = (torch.cuda.mem_get_info(dev)[0] if torch.device(dev).type == "cuda"
                else float("inf"))
        if 8 * (fst + 2 * front_max + xs_sz) > free:
            raise NotImplementedError(
                f"multifrontal {what}: factors need {8 * fst / 1e9:.1f} GB + fronts "
                f"{8 * front_max / 1e9:.1f} GB, {free / 1e9:.1f} GB of HBM free "
                f"({self.total} unknowns)")
        self.F = torch.zeros(max(fst, 1), dtype=F64, device=dev)
        def offsets(sz):  # exclusive prefix sums in (height, id) order
            o = np.zeros(nn, np.int64)
            o[order] = np.cumsum(sz[order]) - sz[order]
            return o

        w_off, y_off, c_off = offsets(pn + bn), offsets(pn), offsets(bn)
        px_off, bx_off = y_off.copy(), c_off.copy()

        # ---- numeric factorization, height by height ---------------------
        a_node = np.minimum(owner[G.a_row], owner[G.a_col]) if len(G.a_row) else G.a_row
        N = int(N)
        vblk = val_t.view(-1, N, N)
        # symmetric diagonal (Jacobi) equilibration, A_s = S A S with
        # S = |diag A|^-1/2 -- SuperLU equilibrates too (splu's default
        # Equil option); it keeps the per-front pivoting of the jump-
        # coefficient operators (mu ratio 1000) as accurate as global
        # partial pivoting.  x = S A_s^-1 S b: S is folded into the gather
        # and the final write of the solve.
        isd = G.a_row == G.a_col
        dvert = np.full(nv, -1, np.int64)
        dvert[G.a_row[isd]] = G.a_k[isd]
        scale = torch.ones(nv * m, dtype=F64, device=dev)
        if equilibrate and nv:
            has = np.flatnonzero(dvert >= 0)
            dg = torch.diagonal(vblk[torch.from_numpy(dvert[has]).to(dev)], dim1=1,
                                dim2=2)[:, :m].abs()
            sc = torch.where(dg > 0, dg.rsqrt(), torch.ones_like(dg))
            scale.view(nv, m)[torch.from_numpy(has).to(dev)] = sc
        scale_h = scale.cpu().numpy()
        a_h = height[a_node] if len(a_node) else a_node
        fronts = {}  # h -> flat tensor;  node -> (h, base, stride)
        fbase = np.zeros(nn, np.int64)
        fstride = pp + bp
        cpad = pp.copy()          # pivot padding of a child's stored Schur complement
        ckey = height.copy()      # fronts[] key of a child's stored Schur complement
        # extend-add on the device (xdg_mf_extend_add) or, XDG_MF_EXTEND=torch
        # / host plans, by per-child indexed adds (bit-identical)
        ext_kernel = (ctx is not None and torch.device(dev).type == "cuda"
                      and os.environ.get("XDG_MF_EXTEND", "kernel") == "kernel")
        if self.comm is not None and not ext_kernel:
            raise NotImplementedError("the multi-GPU factorization needs the device extend-add")
        bad_nodes, dev_perms = [], []
        xpos = {int(t): i for i, t in enumerate(self.xroot)}
        xsend = {}  # this rank's cross-rank roots' Schur complements, by front id
        for pass_buckets in (buckets, buckets_sh):
            if not pass_buckets:
                continue
            in_pass = np.zeros(nn, bool)
            for ts in pass_buckets.values():
                in_pass[ts] = True
            last_use = np.full(H, -1, np.int64)
            tp = np.flatnonzero(in_pass & (parent >= 0))
            tp = tp[in_pass[parent[tp]]]
            if len(tp):
                np.maximum.at(last_use, height[tp], height[parent[tp]])
            for h in range(H):
                hb = [(k, ts) for k, ts in pass_buckets.items() if k[0] == h]
                if not hb:
                    for hh in range(h + 1):
                        if hh in fronts and last_use[hh] <= h:
                            del fronts[hh]
                    continue
                size = 0
                for (_, P_, B_), ts in hb:
                    fbase[ts] = size + np.arange(len(ts)) * (P_ + B_) ** 2
                    size += len(ts) * (P_ + B_) ** 2
                flat = torch.zeros(max(size, 1), dtype=F64, device=dev)
                fronts[h] = flat
                # identity on the pivot padding
                pad_idx = []
                for (_, P_, B_), ts in hb:
                    ts_ = np.asarray(ts, np.int64)
                    ts_ = ts_[pn[ts_] < P_]
                    if len(ts_):
                        i = _ranges(pn[ts_], np.full(len(ts_), P_, np.int64))
                        pad_idx.append(np.repeat(fbase[ts_], P_ - pn[ts_]) + i * (P_ + B_ + 1))
                if pad_idx:
                    flat[torch.from_numpy(np.concatenate(pad_idx)).to(dev)] = 1.0
                # original entries whose earlier-eliminated end is a front of h
                sel = np.flatnonzero((a_h == h) & in_pass[a_node]) if len(a_node) else a_node
                if sel.size:
                    nd_ = a_node[sel]
                    rpos = front_pos(nd_, G.a_row[sel])
                    cpos = front_pos(nd_, G.a_col[sel])
                    # one upload of the per-entry scalars; the m x m target
                    # indices are expanded on the device (on the host they were
                    # nnzb m^2 int64 words: 1.5 GB built and copied at cfg4 size)
                    ent = torch.from_numpy(np.stack(
                        [fbase[nd_] + rpos * fstride[nd_] + cpos, fstride[nd_], G.a_k[sel],
                         G.a_row[sel], G.a_col[sel]])).to(dev)
                    am_d = torch.arange(m, device=dev)
                    tgt = (ent[0][:, None, None] + am_d[None, :, None] * ent[1][:, None, None]
                           + am_d[None, None, :])
                    blocks = vblk[ent[2]][:, :m, :m].transpose(1, 2)
                    sr = scale.view(nv, m)[ent[3]]
                    scl = scale.view(nv, m)[ent[4]]
                    blocks = blocks * sr[:, :, None] * scl[:, None, :]
                    flat[tgt.reshape(-1)] = blocks.reshape(-1)
                    del ent, tgt, blocks, sr, scl
                # children's Schur complements (extend-add), child by child
                if ext_kernel:
                    self._extend_add(ctx, hb, parent, bn, cpad, fbase, fstride, ckey, fronts,
                                     flat, B_list, front_pos, m)
                for t in (() if ext_kernel else (t for (_, _, _), ts in hb for t in ts)):
                    if not kids[t]:
                        continue
                    Ft = flat[fbase[t]:fbase[t] + fstride[t] ** 2].view(fstride[t], fstride[t])
                    for c in kids[t]:
                        if bn[c] == 0:
                            continue
                        fc = fronts[int(height[c])]
                        sc = fstride[c]
                        S = fc[fbase[c]:fbase[c] + sc * sc].view(sc, sc)[
                            pp[c]:pp[c] + bn[c], pp[c]:pp[c] + bn[c]]
                        U = (front_pos(np.full(len(B_list[c]), t), B_list[c])[:, None]
                             + np.arange(m)[None, :]).reshape(-1)
                        Ut = torch.from_numpy(U).to(dev)
                        Ft[Ut[:, None], Ut[None, :]] += S
                # factor every bucket of this height
                for (_, P_, B_), ts in hb:
                    nb = len(ts)
                    n_ = P_ + B_
                    Fb = flat[fbase[ts[0]]:fbase[ts[0]] + nb * n_ * n_].view(nb, n_, n_)
                    if P_ == 0:
                        continue
                    # partial LU of every front of the bucket in place
                    # (xdg_batched_factor, p = P_ of n = P_ + B_ columns): L_BP,
                    # U_PB, the Schur complement for the parent and the
                    # triangular inverses of the pivot block, no library calls
                    if front_factor is not None:  # CPU planning tests (tests/mf_emulation.py)
                        perm, bad = front_factor(Fb, P_)
                    else:
                        foff = fbase[ts[0]] + np.arange(nb, dtype=np.int64) * n_ * n_
                        perm, _, info = batched_factor(
                            ctx, flat, foff, np.full(nb, n_, np.int32),
                            np.full(nb, P_, np.int32), invert=True,
                            perm_off=np.arange(nb, dtype=np.int64) * P_)
                        perm = perm[:nb * P_].view(nb, P_)
                        bad = info[:nb] != 0
                    is_col = bool(colf[ts[0]])
                    if B_:
                        LBP = Fb[:, P_:, :P_]
                        bad |= ~torch.isfinite(LBP).flatten(1).all(1)
                        o, o2 = int(lbp_off[ts[0]]), int(upb_off[ts[0]])
                        out_m = (torch.empty(nb, B_, P_, dtype=F64, device=dev) if is_col
                                 else self.F[o:o + nb * B_ * P_].view(nb, B_, P_))
                        out_n = self.F[o2:o2 + nb * P_ * B_].view(nb, P_, B_)
                        if not merged:
                            out_m.copy_(LBP)
                            out_n.copy_(Fb[:, :P_, P_:])
                        elif front_factor is not None:  # CPU planning tests
                            INV = Fb[:, :P_, :P_]
                            eye = torch.eye(P_, dtype=F64)
                            out_m.copy_(LBP @ (torch.tril(INV, -1) + eye))
                            out_n.copy_(torch.triu(INV) @ Fb[:, :P_, P_:])
                        else:  # M = L_BP L^-1, N = U^-1 U_PB (xdg_mf_merge)
                            for q0 in range(0, nb, 65535):
                                q1 = min(nb, q0 + 65535)
                                nat.check(ctx.lib.xdg_mf_merge(
                                    q1 - q0, P_, B_, Fb[q0:q1].data_ptr(),
                                    out_m[q0:q1].data_ptr(), out_n[q0:q1].data_ptr(),
                                    ctx.stream), "mf_merge")
                    o = int(inv_off[ts[0]])
                    self.F[o:o + nb * P_ * P_].view(nb, P_, P_).copy_(Fb[:, :P_, :P_])
                    if is_col:  # FT[k][r] = [strict-lower L^-1; M_BP][r][k]
                        ld_ = int(ldr[ts[0]])
                        ft = self.F[int(lbp_off[ts[0]]):][:nb * P_ * ld_].view(nb, P_, ld_)
                        ft[:, :, :P_].copy_(torch.tril(Fb[:, :P_, :P_], -1).transpose(1, 2))
                        if B_:
                            ft[:, :, P_:P_ + B_].copy_(out_m.transpose(1, 2))
                    bad_nodes.append((ts, bad))
                    dev_perms.append((ts, perm))  # read back once, after all heights
                    for q, t in enumerate(ts if xpos else ()):  # Schur complements other ranks need
                        if t in xpos:
                            b_ = int(bn[t])
                            xsend[int(t)] = Fb[q, P_:P_ + b_, P_:P_ + b_].reshape(-1).clone()
                for hh in range(h + 1):
                    if hh in fronts and last_use[hh] <= h:
                        del fronts[hh]
            fronts.clear()
            if pass_buckets is buckets and self.comm is not None:
                # every rank receives every cross-rank root's Schur complement
                # (rank order, then id: the xroot order) for the replicated
                # top fronts; they are read in place by the extend-add
                per_rank = [int(sum(int(bn[t]) ** 2 for t in self.xroot
                                    if self.rank_of[t] == r)) for r in range(self.comm.world)]
                # sent in xroot order (the fronts were factored height by height)
                mine_t = [int(t) for t in self.xroot if int(t) in xsend]
                mine = (torch.cat([xsend[t] for t in mine_t]) if mine_t
                        else torch.zeros(0, dtype=F64, device=dev))
                recv = self.comm.allgather_cat(mine, per_rank)
                off = 0
                for t in self.xroot:
                    fbase[t], fstride[t], cpad[t], ckey[t] = off, int(bn[t]), 0, -1
                    off += int(bn[t]) ** 2
                fronts[-1] = recv
                del xsend
        if bad_nodes:
            flags = torch.cat([b.reshape(-1) for _, b in bad_nodes]).cpu().numpy()
            allts = [t for ts, _ in bad_nodes for t in ts]
            if flags.any():
                t = allts[int(np.flatnonzero(flags)[0])]
                blk = tuple(int(b) for b in G.gblk[P_list[t][:8]])
                raise SingularSystemError(f"{what} is singular (front on blocks {blk}...)")
        # pivot permutations of all fronts, laid out front after front in id
        # order (front t at pu_off[t]: position i <- front unknown pu_all[..+i])
        pu_off = np.concatenate([[0], np.cumsum(pn)])
        pu_all = np.zeros(int(pu_off[-1]), np.int64)
        for ts, perm in dev_perms:
            ph = perm.cpu().numpy().astype(np.int64)
            ts_ = np.asarray(ts, np.int64)
            keep = np.arange(ph.shape[1])[None, :] < pn[ts_][:, None]
            pu_all[(pu_off[ts_][:, None] + np.arange(ph.shape[1])[None, :])[keep]] = ph[keep]
        fronts.clear()
        t2 = time.perf_counter()

        # ---- solve plan ---------------------------------------------------
        am = np.arange(m)
        vsrc = np.asarray(vsrc, np.int64)
        vdst = np.asarray(vdst, np.int64)
        # gather entries, node by node in (height, id) order
        # (multi-GPU: entries and tasks of the owned fronts first, then of the
        # shared top fronts -- two sweeps over the heights, self.lev_*[k])
        classes = [need & ~shared, need & shared]
        # (vectorised over all fronts: a Schwarz plan of 337 systems has
        # ~27,000 of them, and per-front numpy calls cost 1 s of its setup)
        Plen, Blen, Pcat = Plen0, Blen0, Pcat0
        Pptr = np.concatenate([[0], np.cumsum(Plen)])
        Bptr = np.concatenate([[0], np.cumsum(Blen)])
        Bcat = bkey_v
        node_of_P = np.repeat(np.arange(nn), Plen)
        node_of_B = bkey_node
        seq = np.concatenate([order[cls[order]] for cls in classes]) if nn else order
        lev_ent_k = []
        ent_first = np.zeros(nn, np.int64)  # first entry id of each node
        cnt_seq = (pn + bn)[seq]
        ent_first[seq] = np.cumsum(cnt_seq) - cnt_seq
        cur = 0
        for cls in classes:
            hs = height[order[cls[order]]]
            sz = (pn + bn)[order[cls[order]]]
            per_h = np.bincount(hs, weights=sz, minlength=H).astype(np.int64) if H else \
                np.zeros(0, np.int64)
            lev_ent_k.append([int(v) for v in cur + np.concatenate([[0], np.cumsum(per_h)])])
            cur += int(sz.sum())
        E = cur
        # permuted pivot unknowns of every needed front, fronts in id order:
        # position i of front t holds front unknown perms[t][i]
        ids = np.flatnonzero(need)
        pu_glob = (pu_all[_ranges(pu_off[ids], pu_off[ids] + pn[ids])]
                   + np.repeat(Pptr[ids] * m, pn[ids]))
        loc = _ranges(np.zeros(len(ids), np.int64), pn[ids])  # i within the front
        inv_perm_all = np.zeros(int(Pptr[-1]) * m, np.int64)  # front unknown -> position
        inv_perm_all[pu_glob] = loc
        src_all = (vsrc[Pcat][:, None] + am[None, :]).reshape(-1)
        scl_all = scale_h.reshape(nv, m)[Pcat].reshape(-1)
        ent_src = np.full(E, -1, np.int64)
        ent_scale = np.ones(E)
        piv_ent = np.repeat(ent_first[ids], pn[ids]) + loc
        ent_src[piv_ent] = src_all[pu_glob]
        ent_scale[piv_ent] = scl_all[pu_glob]
        ent_w = _ranges(w_off[seq], w_off[seq] + cnt_seq)
        # contributions: child c's boundary unknown j -> parent's entry
        par_B = parent[node_of_B] if nn else node_of_B
        okc = (par_B >= 0) & need[np.maximum(par_B, 0)] if nn else np.zeros(0, bool)
        cB, tB, vB = node_of_B[okc], par_B[okc], Bcat[okc]
        jB = (np.arange(len(Bcat)) - Bptr[node_of_B])[okc]  # position in the child's B
        inP = owner[vB] == tB
        fu0 = np.empty(len(vB), np.int64)  # unpermuted front unknown (mode 0)
        fu0[inP] = ppos[vB[inP]] * m
        fu0[~inP] = pn[tB[~inP]] + bpos(tB[~inP], vB[~inP]) * m
        fu = (fu0[:, None] + am[None, :]).reshape(-1)
        tt = np.repeat(tB, m)
        piv = fu < pn[tt]
        ent = fu.copy()
        ent[piv] = inv_perm_all[Pptr[tt[piv]] * m + fu[piv]]
        c_tgt = ent_first[tt] + ent
        c_src = ((c_off[cB] + jB * m)[:, None] + am[None, :]).reshape(-1)
        if len(c_tgt):
            so = np.argsort(c_tgt, kind="stable")  # children in id order per entry
            c_tgt, c_src = c_tgt[so], c_src[so]
        ent_cptr = np.zeros(len(ent_w) + 1, np.int64)
        np.cumsum(np.bincount(c_tgt, minlength=len(ent_w)), out=ent_cptr[1:])
        # warp tasks, level-sorted: (node, first row), 32/G rows each
        gp = _group_v(pn)
        gb = np.where(bn > 0, _group_v(bn), gp)
        if merged:  # a backward row = U^-1 row (<= p long) + N_PB row (b long)
            gb = np.maximum(gp, gb)

        def tasks(phase, cls):
            """int4 warp tasks (node, first row, rows, -1) of one phase, level
            by level: fronts whose rows take a whole warp (G = 32) get MR rows
            per task; shorter rows 32/G rows per task (rows field 0)."""
            g = gb if phase == 2 else gp
            nrows = bn if phase == 1 else pn
            if merged:
                g = gb if phase in (2, 3) else gp
            if merged:  # phases 0, 1: forward rows 0..p+b-1; 2, 3: backward rows
                nrows = pn + bn if phase in (0, 1) else pn
            out, lev = [], []
            for h in range(H):
                ts = order[(height[order] == h) & cls[order]]
                if merged and phase == 4:  # one thread per forward row
                    cf = ts[colf[ts]]
                    cnt = (pn[cf] + bn[cf] + 31) // 32
                    first = _ranges(np.zeros(len(cf), np.int64), cnt) * 32
                    ct_ = np.stack([np.repeat(cf, cnt), first, np.full_like(first, -3),
                                    np.full_like(first, -1)], 1)
                    out.append(ct_)
                    lev.append(len(ct_))
                    continue
                if merged and phase == 5:
                    lev.append(0)
                    continue
                if merged and phase in (0, 1):
                    ts = ts[~colf[ts]]
                if merged:
                    # whole-warp fronts: MR rows per task; rows of >= LONG
                    # elements are CTA tasks (slots 1 / 3), the others warp
                    # tasks (slots 0 / 2), which also hold the short fronts
                    lg = ts[g[ts] == 32]
                    cnt2 = (nrows[lg] + MR - 1) // MR
                    r2 = _ranges(np.zeros(len(lg), np.int64), cnt2) * MR
                    node2 = np.repeat(lg, cnt2)
                    if phase in (0, 1):  # longest row of the task: r + MR - 1 or p
                        ln = np.minimum(r2 + MR - 1, pn[node2])
                    else:
                        ln = pn[node2] - r2 + bn[node2]
                    # group tasks only where the warp tasks would not fill
                    # the GPU a few times over (a barrier per task costs ~10 %)
                    if len(r2) >= WAVES * RESIDENT_WARPS:
                        ln = np.zeros_like(ln)
                    pick = (ln >= LONG) if phase in (1, 3) else (ln < LONG)
                    long_ = np.stack([node2[pick], r2[pick], np.full(int(pick.sum()), MR),
                                      np.full(int(pick.sum()), -1)], 1)
                    if phase in (1, 3):
                        out.append(long_)
                        lev.append(len(long_))
                        continue
                    sh = ts[g[ts] < 32]
                    per = (32 // g[sh]) * 2
                    cnt = (nrows[sh] + per - 1) // per
                    first = _ranges(np.zeros(len(sh), np.int64), cnt) * np.repeat(per, cnt)
                    grp = np.stack([np.repeat(sh, cnt), first, np.full_like(first, -2),
                                    np.full_like(first, -1)], 1)
                    out += [grp, long_]
                    lev.append(len(grp) + len(long_))
                    continue
                sh = ts[g[ts] < 32]
                # bound / upb rows all span the same columns: two row sets
                # per task share the vector loads (kernel: group_dot2)
                sets = 2 if merged else (SETS if phase in (1, 2) else 1)
                per = (32 // g[sh]) * sets
                cnt = (nrows[sh] + per - 1) // per
                first = _ranges(np.zeros(len(sh), np.int64), cnt) * np.repeat(per, cnt)
                grp = np.stack([np.repeat(sh, cnt), first,
                                np.full_like(first, 0 if sets == 1 else -2),
                                np.full_like(first, -1)], 1)
                lg = ts[g[ts] == 32]
                cnt2 = (nrows[lg] + MR - 1) // MR
                r2 = _ranges(np.zeros(len(lg), np.int64), cnt2) * MR
                long_ = np.stack([np.repeat(lg, cnt2), r2, np.full_like(r2, MR),
                                  np.full_like(r2, -1)], 1)
                out += [grp, long_]
                lev.append(len(grp) + len(long_))
            return out, lev

        MR = _rows_per_warp()
        SETS = _row_sets()
        LONG = _long_row()
        import os as _os
        WAVES = float(_os.environ.get("XDG_MF_CTA_WAVES", "3.0"))
        # group tasks where a launch has fewer than WAVES x 3,552 warp tasks (a
        # measured threshold: 2,368 / 4,736 / 7,104 -> 2.33 / 2.23 / 2.23 ms with
        # the current row kernels, profiles/r2_mf_mr3_waves.txt).  The split
        # decides the summation order of the long rows, i.e. the roundoff: at
        # cfg2 the GMRES count at the 1e-10 floor moved between 6,774 and 8,422
        # over the settings of profiles/r2_gmres_cfg2_split_counts.txt
        RESIDENT_WARPS = 148 * 24
        all_tasks, lev_task_k = [], []
        base = 0
        for cls in classes:
            lev_task = []
            for phase in range(6 if merged else 4):
                tl, lv = tasks(phase, cls)
                all_tasks += tl
                lev_task.append(base + np.concatenate([[0], np.cumsum(lv)]))
                base += int(np.sum(lv))
            lev_task_k.append(lev_task)
        task_arr = (np.concatenate(all_tasks) if all_tasks
                    else np.zeros((0, 4), np.int64))
        lev_task = lev_task_k[0]
        lev_ent = lev_ent_k[0]
        self._fused_plan(task_arr, lev_task, ent_first, pn, bn, height, parent, order, H,
                         off=self.comm is not None or merged)
        bidx = np.zeros(int(bn.sum()), np.int64)
        pdst = np.zeros(int(pn.sum()), np.int64)
        pscale = np.ones(int(pn.sum()))
        if nn:
            # Y position (owner's pivot space) of each boundary unknown
            jB_all = np.arange(len(Bcat)) - Bptr[node_of_B]
            bpos_all = ((c_off[node_of_B] + jB_all * m)[:, None] + am[None, :]).reshape(-1)
            bidx[bpos_all] = ((y_off[owner[Bcat]] + ppos[Bcat] * m)[:, None]
                              + am[None, :]).reshape(-1)
            jP_all = np.arange(len(Pcat)) - Pptr[node_of_P]
            ppos_all = ((y_off[node_of_P] + jP_all * m)[:, None] + am[None, :]).reshape(-1)
            pdst[ppos_all] = (vdst[Pcat][:, None] + am[None, :]).reshape(-1)
            pscale[ppos_all] = scl_all
        nodes = np.zeros(nn, NODE_DT)
        nodes["p"], nodes["b"], nodes["ldp"], nodes["ldb"] = pn, bn, pp, bp
        nodes["gp"], nodes["gb"] = gp, gb
        nodes["ldr"] = ldr  # leading dimension of the column-major forward copy
        nodes["inv"], nodes["lbp"], nodes["upb"] = inv_off, lbp_off, upb_off
        nodes["w"], nodes["y"], nodes["c"] = w_off, y_off, c_off
        nodes["bx"], nodes["px"] = bx_off, px_off

        def up(a, dt):
            return torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt)

        self.lev_ent = np.asarray(lev_ent, np.int64)
        self.lev_task = np.ascontiguousarray(np.concatenate(lev_task), np.int64)
        # second sweep (shared top fronts, multi-GPU only)
        self.lev_ent_sh = np.asarray(lev_ent_k[1], np.int64)
        self.lev_task_sh = np.ascontiguousarray(np.concatenate(lev_task_k[1]), np.int64)
        self.task_host = task_arr
        self.ent_w, self.ent_src = up(ent_w, I64), up(ent_src, I64)
        self.ent_cptr, self.ent_cidx = up(ent_cptr, I64), up(c_src, I64)
        self.tasks = up(task_arr, I32)
        self.nodes_host = nodes
        self.nodes = torch.from_numpy(nodes.view(np.uint8).copy()).to(dev)
        self.bidx, self.pdst = up(bidx, I64), up(pdst, I64)
        self.ent_scale, self.pscale = up(ent_scale, F64), up(pscale, F64)
        self.W = torch.zeros(max(int((pn + bn).sum()), 1), dtype=F64, device=dev)
        self.Y = torch.zeros(max(int(pn.sum()), 1), dtype=F64, device=dev)
        self.C = torch.zeros(max(int(bn.sum()), 1), dtype=F64, device=dev)
        self.X = torch.zeros(max(int(pn.sum()), 1) if merged else 1, dtype=F64, device=dev)
        self.factor_bytes = 8 * int((pn * pn + 2 * pn * bn)[need].sum())
        self.apply_bytes = self.factor_bytes + 8 * int(4 * (pn + bn)[need].sum()
                                                       + 4 * pn[need].sum())
        if self.comm is not None:
            self._dist_plan(pn, bn, c_off, y_off, vdst, P_list, am, dev)
        self.pn, self.bn = pn, bn
        self.colf = colf
        self._s = None
        self.times = {"symbolic": t1 - t0, "numeric": t2 - t1,
                      "plan": time.perf_counter() - t2}

    # ------------------------------------------------------------------
    @staticmethod
    def _extend_add(ctx, hb, parent, bn, pp, fbase, fstride, height, fronts, flat, B_list,
                    front_pos, m):
        """Device extend-add of one height (xdg_mf_extend_add): round r adds
        the r-th child (ascending id = kids order, bn > 0) of every parent, one
        launch per (round, child height).  Array operations over all the
        (parent, child) pairs of the height."""
        nn = len(parent)
        in_h = np.zeros(nn, bool)
        for (_, _, _), ts in hb:
            in_h[ts] = True
        cc_all = np.flatnonzero((parent >= 0) & (bn > 0))
        cc_all = cc_all[in_h[parent[cc_all]]]
        if not len(cc_all):
            return
        so = np.argsort(parent[cc_all], kind="stable")  # children ascending per parent
        cc_all = cc_all[so]
        tt_all = parent[cc_all]
        first = np.concatenate([[True], tt_all[1:] != tt_all[:-1]])
        start = np.maximum.accumulate(np.where(first, np.arange(len(tt_all)), 0))
        rnd = np.arange(len(tt_all)) - start
        Bflat, Blen = _flat(B_list)
        Bptr = np.concatenate([[0], np.cumsum(Blen)])
        key = rnd * (int(height.max()) + 2) + (height[cc_all] + 1)  # ckey may be -1
        dev = flat.device
        for k in np.unique(key):
            selk = key == k
            tt, cc = tt_all[selk], cc_all[selk]
            nodes_ = np.repeat(tt, Blen[cc])
            verts = Bflat[_ranges(Bptr[cc], Bptr[cc + 1])]
            U = (front_pos(nodes_, verts)[:, None] + np.arange(m)[None, :]).reshape(-1)
            n = bn[cc].astype(np.int64)
            uoff = np.concatenate([[0], np.cumsum(n)[:-1]])
            pair = np.stack([fbase[tt], fstride[tt], fbase[cc], fstride[cc], pp[cc], n, uoff],
                            1).astype(np.int64)
            pair_d = torch.from_numpy(np.ascontiguousarray(pair)).to(dev)
            U_d = torch.from_numpy(np.ascontiguousarray(U, np.int64)).to(dev)
            child = fronts[int(height[cc[0]])]
            nat.check(ctx.lib.xdg_mf_extend_add(len(tt), pair_d.data_ptr(), U_d.data_ptr(),
                                                child.data_ptr(), flat.data_ptr(),
                                                int(n.max()), ctx.stream), "mf_extend_add")

    def _fused_plan(self, task_arr, lev_task, ent_first, pn, bn, height, parent, order, H,
                    off=False):
        """Groups / stages of the fused low levels (XDG_MF_FUSE).  A stage is
        a set of fronts of one height; its gather entries and its warp tasks
        of each phase are copied out stage by stage (the same int4 tasks the
        per-level launches run)."""
        mode, K = _fuse_mode()
        K = 0 if off else min(K, H)
        nn = len(pn)
        dev = self.F.device
        if K == 0:
            self.fuse_levels = self.nfbatch = self.nfstages = 0
            self.fb_grp = np.zeros(1, np.int64)
            self.g_stage = self.st_ent = self.st_task = self.fent = torch.zeros(
                1, dtype=I64, device=dev)
            self.ftask = torch.zeros(4, dtype=I32, device=dev)
            return
        # per-node warp-task range of each phase (tasks of a node contiguous)
        trng = []
        for ph in range(4):
            a, e = int(lev_task[ph][0]), int(lev_task[ph][-1])
            nodes_ = task_arr[a:e, 0]
            st = np.full(nn, 0, np.int64)
            ct = np.bincount(nodes_, minlength=nn).astype(np.int64)
            if len(nodes_):
                chg = np.flatnonzero(np.r_[True, nodes_[1:] != nodes_[:-1]])
                assert len(chg) == int((ct > 0).sum()), "tasks of a node not contiguous"
                st[nodes_[chg]] = a + chg
            trng.append((st, ct))
        groups = []  # per batch: list of groups; group = list of stages (node arrays)
        if K > 0 and mode == "level":
            for h in range(K):
                ts = order[height[order] == h]
                groups.append([[np.array([t])] for t in ts])
        elif K > 0:
            low = height < K
            root = np.arange(nn)
            top = low & ((parent < 0) | ~low[np.maximum(parent, 0)])
            # root of every low node (post-order: ids increase toward the root)
            for t in range(nn - 1, -1, -1):
                if low[t] and not top[t]:
                    root[t] = root[parent[t]]
            batch = []
            members = {}
            for t in order:  # by height, then id
                if low[t]:
                    members.setdefault(int(root[t]), []).append(int(t))
            for r in sorted(members, key=lambda r: (-height[r], r)):
                ms = np.array(members[r], np.int64)
                batch.append([ms[height[ms] == h] for h in range(int(height[r]) + 1)])
            groups.append(batch)
        fb_grp, g_stage, st_ent, fent = [0], [0], [0], []
        st_task = [[0] for _ in range(4)]
        ftask = [[] for _ in range(4)]
        tcount = [0, 0, 0, 0]
        for batch in groups:
            for grp in batch:
                for nodes_ in grp:
                    e = [np.arange(ent_first[t], ent_first[t] + pn[t] + bn[t]) for t in nodes_]
                    fent += e
                    st_ent.append(st_ent[-1] + sum(len(x) for x in e))
                    for ph in range(4):
                        st, ct = trng[ph]
                        for t in nodes_:
                            if ct[t]:
                                ftask[ph].append(task_arr[st[t]:st[t] + ct[t]])
                                tcount[ph] += int(ct[t])
                        st_task[ph].append(tcount[ph])
                g_stage.append(len(st_ent) - 1)
            fb_grp.append(len(g_stage) - 1)
        ns = len(st_ent) - 1
        base = np.cumsum([0] + tcount[:3])
        st_task = np.concatenate([np.asarray(st_task[ph], np.int64) + base[ph]
                                  for ph in range(4)])
        ft = [np.concatenate(ftask[ph]) for ph in range(4) if ftask[ph]]
        ft = np.concatenate(ft) if ft else np.zeros((1, 4), np.int64)
        fe = np.concatenate(fent) if fent else np.zeros(1, np.int64)
        self.fuse_levels = K if groups else 0
        self.nfbatch, self.nfstages = len(groups), ns
        self.fb_grp = np.asarray(fb_grp, np.int64)
        self.g_stage = torch.tensor(g_stage, dtype=I64, device=dev)
        self.st_ent = torch.tensor(st_ent, dtype=I64, device=dev)
        self.st_task = torch.from_numpy(st_task).to(dev)
        self.fent = torch.from_numpy(np.ascontiguousarray(fe, np.int64)).to(dev)
        self.ftask = torch.from_numpy(np.ascontiguousarray(ft)).to(dev, I32)

    def _dist_plan(self, pn, bn, c_off, y_off, vdst, P_list, am, dev):
        """Index lists of the two exchanges of a multi-GPU solve: the
        contributions C of the cross-rank subtree roots (after the owned
        forward sweep) and the solution entries of every rank's owned fronts
        (after the owned backward sweep), both in (rank, front id) order."""
        comm, me = self.comm, self.comm.rank
        W = comm.world

        def pack(sel_fronts, rng):
            per, mine, allv = [], None, []
            for r in range(W):
                ts = [t for t in sel_fronts if self.rank_of[t] == r]
                idx = (np.concatenate([rng(t) for t in ts]) if ts
                       else np.zeros(0, np.int64))
                per.append(len(idx))
                allv.append(idx)
                if r == me:
                    mine = idx
            up = (lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32)).to(dev))
            return per, up(mine), up(np.concatenate(allv))

        self.xc_counts, self.xc_mine, self.xc_all = pack(
            list(self.xroot), lambda t: c_off[t] + np.arange(bn[t]))
        owned = [t for t in range(len(pn)) if self.rank_of[t] >= 0 and pn[t] > 0]
        self.xo_counts, self.xo_mine, self.xo_all = pack(
            owned, lambda t: (vdst[P_list[t]][:, None] + am).reshape(-1))
        self.xc_send = torch.empty(max(len(self.xc_mine), 1), dtype=F64, device=dev)
        self.xo_send = torch.empty(max(len(self.xo_mine), 1), dtype=F64, device=dev)

    def struct(self, shared: bool = False) -> XdgMf:
        if shared:  # the replicated top fronts' sweep (multi-GPU)
            if getattr(self, "_s_sh", None) is None:
                s = XdgMf()
                C.memmove(C.addressof(s), C.addressof(self.struct()), C.sizeof(XdgMf))
                s.lev_ent = self.lev_ent_sh.ctypes.data
                s.lev_task = self.lev_task_sh.ctypes.data
                s.fuse_levels = s.nfbatch = 0
                self._s_sh = s
            return self._s_sh
        if self._s is None:
            s = XdgMf()
            s.nlevels, s.nnodes, s.total = self.nlevels, self.nnodes, self.total
            s.lev_ent = self.lev_ent.ctypes.data
            s.lev_task = self.lev_task.ctypes.data
            for f in ("ent_w", "ent_src", "ent_cptr", "ent_cidx", "tasks", "nodes",
                      "ent_scale", "pscale", "bidx", "pdst", "F", "W", "Y", "C"):
                setattr(s, f, getattr(self, f).data_ptr())
            s.apply_bytes = float(self.apply_bytes)
            s.fuse_levels, s.nfbatch, s.nfstages = self.fuse_levels, self.nfbatch, self.nfstages
            s.fb_grp = self.fb_grp.ctypes.data
            for f in ("g_stage", "st_ent", "st_task", "fent", "ftask"):
                setattr(s, f, getattr(self, f).data_ptr())
            s.X, s.merged = self.X.data_ptr(), int(self.merged)
            self._s = s
        return self._s

    def solve(self, b: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        """x[vdst + a] = A^-1 b[vsrc + a] for every system (device tensors).
        Multi-GPU: every rank passes the whole b and receives the whole x;
        it sweeps its owned subtrees and the replicated top fronts, with one
        all-gather of the subtree roots' contributions in between and one of
        the owned fronts' solution entries at the end."""
        lib, st = self.ctx.lib, self.ctx.stream
        if self.comm is None:
            nat.check(lib.xdg_mf_solve(C.byref(self.struct()), b.data_ptr(), x.data_ptr(), st),
                      "mf_solve")
            return x
        nat.check(lib.xdg_mf_solve_phase(C.byref(self.struct()), b.data_ptr(), x.data_ptr(),
                                         1, st), "mf_solve(owned forward)")
        self._exchange(self.C, self.xc_mine, self.xc_all, self.xc_counts, self.xc_send)
        nat.check(lib.xdg_mf_solve_phase(C.byref(self.struct(True)), b.data_ptr(),
                                         x.data_ptr(), 3, st), "mf_solve(shared)")
        nat.check(lib.xdg_mf_solve_phase(C.byref(self.struct()), b.data_ptr(), x.data_ptr(),
                                         2, st), "mf_solve(owned backward)")
        self._exchange(x, self.xo_mine, self.xo_all, self.xo_counts, self.xo_send)
        return x

    def _exchange(self, buf, mine, allv, counts, send):
        """buf[allv] = concatenation over ranks of buf_r[mine_r]."""
        lib, st = self.ctx.lib, self.ctx.stream
        nat.check(lib.xdg_gather_blocks(len(mine), 1, mine.data_ptr(), buf.data_ptr(),
                                        send.data_ptr(), st), "gather(exchange)")
        recv = self.comm.allgather_cat(send[:len(mine)], counts)
        nat.check(lib.xdg_scatter_blocks(len(allv), 1, allv.data_ptr(), recv.data_ptr(),
                                         buf.data_ptr(), st), "scatter(exchange)")


def _ipiv_to_perm(ctx, piv: torch.Tensor, n: int) -> torch.Tensor:
    """LAPACK ipiv (batch, n) -> row permutation (batch, n), int32."""
    nb = piv.shape[0]
    if piv.is_cuda:
        from .direct import ipiv_to_perm

        dims = torch.full((nb,), n, dtype=I32, device=piv.device)
        off = torch.arange(nb, dtype=I64, device=piv.device) * n
        return ipiv_to_perm(ctx, piv.reshape(-1), dims, off).view(nb, n)
    # host tensors (CPU unit tests of the factorization)
    ip = piv.numpy() - 1
    perm = np.tile(np.arange(n, dtype=np.int32), (nb, 1))
    rows = np.arange(nb)
    for i in range(n):
        j = ip[:, i]
        a, b = perm[rows, i].copy(), perm[rows, j].copy()
        perm[rows, i], perm[rows, j] = b, a
    return torch.from_numpy(perm)
