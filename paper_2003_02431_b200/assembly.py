"""SIP-DG assembly of the two-phase Poisson problem.

Restates cutdg assembly.py:255-422 (assemble_sip / assemble_rhs) in the
plain background basis (basis.py:52-104, no per-piece orthonormalisation --
bench.py:178) with the penalty of assembly.py:133-203.

B200 layout.  On a uniform Cartesian mesh every *regular* contribution --
the volume term of an uncut piece, the interior-face and boundary-face terms
of a face not touched by the interface -- is one of a few reference blocks
scaled by scalars: mu_s * K for volumes, mu * C + (eta mu) * P for faces (C:
consistency + symmetry terms, P: penalty term; per axis and side).  The host
therefore emits, per output block, a list of (table, coefficient) terms plus
the indices of the exact dense blocks of cut items (cut volumes, cut face
portions, interface patches: evaluated per item with the reference's own
operations), and `xdg_assemble_blocks` forms all blocks in HBM, column-major
(BSR-T), in one pass bounded by the output write.  Regular blocks differ from
the reference's per-cell evaluation only by roundoff (the reference evaluates
each cell's basis at its own physical nodes); tests bound the difference at
1e-12 relative.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from functools import lru_cache
from math import comb
from typing import Callable, Optional

import numpy as np

from .cutcells import SPECIES, CutCellMesh, embed, quad_cut_face, quad_volume, tensor_rule
from .errors import InvalidConfigError, MissingSpeciesError
from .geometry import NEG, POS

DIRICHLET, NEUMANN = "dirichlet", "neumann"


# ---------------------------------------------------------------------------
# plain tensor-Legendre basis (basis.py:17-104)

@lru_cache(maxsize=None)
def multi_indices(degree: int, dim: int):
    idx = [b for b in np.ndindex(*([degree + 1] * dim)) if sum(b) <= degree]
    idx.sort(key=lambda b: (sum(b), b))
    return tuple(tuple(int(x) for x in b) for b in idx)


def _legendre_all(t, k):
    vals = np.empty(t.shape + (k + 1,))
    ders = np.empty(t.shape + (k + 1,))
    vals[..., 0] = 1.0
    ders[..., 0] = 0.0
    if k >= 1:
        vals[..., 1] = t
        ders[..., 1] = 1.0
    for n in range(1, k):
        vals[..., n + 1] = ((2 * n + 1) * t * vals[..., n] - n * vals[..., n - 1]) / (n + 1)
        ders[..., n + 1] = ders[..., n - 1] + (2 * n + 1) * vals[..., n]
    return vals, ders


class PlainBasis:
    """Orthonormal (on the full cell) tensor-Legendre basis of total degree
    <= k.  `lo`/`hi` may carry leading batch dimensions matching `points`
    (..., P, D); per element the arithmetic is the reference's."""

    def __init__(self, degree: int, dim: int):
        self.degree, self.dim = int(degree), int(dim)
        self.indices = multi_indices(self.degree, self.dim)
        self.size = len(self.indices)
        assert self.size == comb(self.degree + self.dim, self.dim)
        self._idx = np.array(self.indices)

    def _tables(self, lo, hi, pts):
        pts = np.asarray(pts, float)
        lo = np.asarray(lo, float)[..., None, :]
        hi = np.asarray(hi, float)[..., None, :]
        k = self.degree
        vals, ders = [], []
        for a in range(self.dim):
            width = hi[..., a] - lo[..., a]
            t = (2.0 * pts[..., a] - lo[..., a] - hi[..., a]) / width
            v, d = _legendre_all(t, k)
            norm = np.sqrt((2 * np.arange(k + 1) + 1) / width[..., None])
            vals.append(v * norm)
            ders.append(d * norm * (2.0 / width[..., None]))
        return vals, ders

    def eval(self, lo, hi, pts):
        vals, _ = self._tables(lo, hi, pts)
        out = np.ones(np.shape(pts)[:-1] + (self.size,))
        for a in range(self.dim):
            out *= vals[a][..., self._idx[:, a]]
        return out

    def eval_with_grad(self, lo, hi, pts):
        vals, ders = self._tables(lo, hi, pts)
        shp = np.shape(pts)[:-1] + (self.size,)
        value = np.ones(shp)
        for a in range(self.dim):
            value *= vals[a][..., self._idx[:, a]]
        grad = np.empty(shp + (self.dim,))
        for g in range(self.dim):
            comp = np.ones(shp)
            for a in range(self.dim):
                comp *= (ders[a] if a == g else vals[a])[..., self._idx[:, a]]
            grad[..., g] = comp
        return value, grad


# ---------------------------------------------------------------------------
# problem and penalty (assembly.py:34-203)

def _zero(points, *_):
    return np.zeros(len(points))


def _one(points, *_):
    return np.ones(len(points))


@dataclass
class PoissonProblem:
    """mu_a on phi < 0 (NEG), mu_b on phi > 0 (POS); `boundary` maps
    (axis, side) -> (kind, g(points[, species]))."""

    mu_a: float
    mu_b: float
    source: Callable = _one
    boundary: dict = field(default_factory=dict)

    def __post_init__(self):
        if not (self.mu_a > 0 and self.mu_b > 0):
            raise InvalidConfigError(
                f"diffusion coefficients must be positive, got {self.mu_a}, {self.mu_b}")

    def mu(self, s):
        return self.mu_a if s == NEG else self.mu_b

    @property
    def mu_max(self):
        return max(self.mu_a, self.mu_b)

    def condition(self, axis, side):
        if (axis, side) not in self.boundary:
            raise InvalidConfigError(f"no boundary condition for domain face {(axis, side)}")
        return self.boundary[(axis, side)]


def dirichlet_problem(mu_a, mu_b, source=_one, dim=3, g=_zero) -> PoissonProblem:
    return PoissonProblem(mu_a, mu_b, source,
                          {(a, s): (DIRICHLET, g) for a in range(dim) for s in (0, 1)})


def _bvals(g, pts, s):
    try:
        return np.asarray(g(pts, s), float)
    except TypeError:
        return np.asarray(g(pts), float)


@dataclass
class PieceIndex:
    """Present pieces in XdgIndexMap order (spaces.py:68-91): cell-major,
    NEG before POS.  block[j, s] = raw block index or -1."""

    pieces: np.ndarray   # (B, 2) int: (cell, species)
    block: np.ndarray    # (J, 2) int

    @classmethod
    def build(cls, species_volume):
        present = species_volume > 0
        block = np.full(present.shape, -1, np.int64)
        block[present] = np.arange(int(present.sum()))
        j, s = np.nonzero(present)
        return cls(np.stack([j, s], axis=1), block)

    @property
    def num_blocks(self):
        return len(self.pieces)


def cell_faces(cm: CutCellMesh) -> np.ndarray:
    """(J, 2D) face ids per cell in fid order: axis0 lo, axis0 hi, ...
    (the order PenaltyScales walks them, assembly.py:145-148)."""
    J, D = cm.num_cells, cm.mesh.dim
    out = np.full((J, 2 * D), -1, np.int64)
    f = cm.faces
    ids = np.arange(len(f))
    for a in range(D):
        on = f.axis == a
        p = on & (f.plus >= 0)
        out[f.plus[p], 2 * a] = ids[p]
        m = on & (f.minus >= 0)
        out[f.minus[m], 2 * a + 1] = ids[m]
    return out


def penalty_inv_h(cm: CutCellMesh, pidx: PieceIndex, groups) -> np.ndarray:
    """1/h' per raw block (PenaltyScales, assembly.py:133-174): aggregate
    surface (outer face portions + all member interface area) over
    D * aggregate volume, with the reference's summation order."""
    D = cm.mesh.dim
    cf = cell_faces(cm)
    f = cm.faces
    fsm = cm.face_species_measure
    im = cm.interface_measures()
    j, s = pidx.pieces[:, 0], pidx.pieces[:, 1]
    # singleton groups, vectorised: area = ((0 + im) + f0) + f1 ...
    area = 0.0 + im[j]
    for q in range(2 * D):
        area = area + fsm[cf[j, q], s]
    inv = area / (D * (0.0 + cm.species_volume[j, s]))
    for g in groups:
        if len(g) == 1:
            continue
        members = set(g)
        vol = 0.0
        ar = 0.0
        for (jj, ss) in g:
            vol += cm.species_volume[jj, ss]
            ar += im[jj]
            for q in range(2 * D):
                fid = cf[jj, q]
                other = f.plus[fid] if f.minus[fid] == jj else f.minus[fid]
                if other < 0 or (int(other), ss) not in members:
                    ar += fsm[fid, ss]
        val = ar / (D * vol)
        for (jj, ss) in g:
            inv[pidx.block[jj, ss]] = val
    return inv


def _stiffness(weights, G):
    """sum_p w_p G_p G_p^T (the einsum "p,pid,pld->il" of assembly.py:275)
    as one GEMM over the (point, axis) pairs."""
    P, N, D = G.shape
    Gt = G.transpose(1, 0, 2).reshape(N, P * D)
    return (Gt * np.repeat(weights, D)[None, :]) @ Gt.T


def _pair_terms(weights, eta, mu_pen, sides):
    """assembly.py:236-252."""
    n = len(sides)
    mean = 1.0 if n == 1 else 0.5
    out = {}
    for a, (Va, Gna, sa) in enumerate(sides):
        Wa = Va * weights[:, None]
        for b, (Vb, Gnb, sb) in enumerate(sides):
            out[(a, b)] = (-mean * sa * Wa.T @ Gnb - mean * sb * (Gna * weights[:, None]).T @ Vb
                           + eta * mu_pen * sa * sb * Wa.T @ Vb)
    return out


# ---------------------------------------------------------------------------
# cut items: per-item dense blocks with the reference's operations

def _eval_item(item):
    from ._pool import STATE

    cm, basis, problem = STATE["cm"], STATE["basis"], STATE["problem"]
    mesh = cm.mesh
    kind = item[0]
    if kind == "vol":
        _, b, j, s = item
        rule = quad_volume(cm, j, s)
        V, G = basis.eval_with_grad(*mesh.bounds(j), rule.nodes)
        return ([(b, b, problem.mu(s) * _stiffness(rule.weights, G))],
                [(b, V.T @ (rule.weights * problem.source(rule.nodes)))])
    if kind == "face":
        _, fid, s, a, jm, jp, bm, bp, eta, mu = item
        rule = quad_cut_face(cm, fid, s)
        Vm, Gm = basis.eval_with_grad(*mesh.bounds(jm), rule.nodes)
        Vp, Gp = basis.eval_with_grad(*mesh.bounds(jp), rule.nodes)
        blocks = _pair_terms(rule.weights, eta, mu,
                             [(Vm, mu * Gm[:, :, a], 1.0), (Vp, mu * Gp[:, :, a], -1.0)])
        idb = (bm, bp)
        return [(idb[x], idb[y], blk) for (x, y), blk in blocks.items()], []
    if kind == "bface":
        _, fid, s, a, side, j, b, eta, mu = item
        bkind, g = problem.condition(a, side)
        sign = -1.0 if side == 0 else 1.0
        rule = quad_cut_face(cm, fid, s)
        V, G = basis.eval_with_grad(*mesh.bounds(j), rule.nodes)
        gv = _bvals(g, rule.nodes, s)
        if bkind == NEUMANN:
            return [], [(b, V.T @ (rule.weights * mu * gv))]
        blk = _pair_terms(rule.weights, eta, mu, [(V, mu * sign * G[:, :, a], 1.0)])
        Gn = sign * G[:, :, a]
        return [(b, b, blk[(0, 0)])], [(b, (eta * V - Gn).T @ (rule.weights * mu * gv))]
    _, j, bn, bp, eta = item
    rule = cm.interface_rules[j]
    Vn, Gn_ = basis.eval_with_grad(*mesh.bounds(j), rule.nodes)
    gn = (Gn_ * rule.normals[:, None, :]).sum(axis=2)
    sides = [(Vn, problem.mu(NEG) * gn, 1.0), (Vn, problem.mu(POS) * gn, -1.0)]
    blocks = _pair_terms(rule.weights, eta, problem.mu_max, sides)
    idb = (bn, bp)
    return [(idb[x], idb[y], blk) for (x, y), blk in blocks.items()], []


def _eval_items(cm, basis, problem, items, workers=None):
    from ._pool import fork_map

    return fork_map(_eval_item, items, dict(cm=cm, basis=basis, problem=problem), workers)


# ---------------------------------------------------------------------------
# term lists

@dataclass
class SipTerms:
    """Raw system in term-list form.  Output blocks (row_ptr, col) in sorted
    (row, col) order; per output o: table terms tptr[o]:tptr[o+1] of
    (tid, coef) and dense terms dptr[o]:dptr[o+1] indexing `dense`.  Tables
    and dense blocks are row-major (N, N)."""

    N: int
    nblocks: int
    row_ptr: np.ndarray
    col: np.ndarray
    tptr: np.ndarray
    tid: np.ndarray
    coef: np.ndarray
    dptr: np.ndarray
    didx: np.ndarray
    tables: np.ndarray
    dense: np.ndarray
    rhs: np.ndarray

    def evaluate_host(self) -> np.ndarray:
        """Row-major values (tests only: the product path is the kernel)."""
        out = np.zeros((len(self.col), self.N, self.N))
        o_t = np.repeat(np.arange(len(self.col)), np.diff(self.tptr))
        np.add.at(out, o_t, self.coef[:, None, None] * self.tables[self.tid])
        o_d = np.repeat(np.arange(len(self.col)), np.diff(self.dptr))
        np.add.at(out, o_d, self.dense[self.didx])
        return out


class _TermBuilder:
    def __init__(self, N):
        self.N = N
        self.tables = []
        self.t_rows, self.t_cols, self.t_tid, self.t_coef = [], [], [], []
        self.d_rows, self.d_cols, self.dense = [], [], []

    def table(self, T):
        self.tables.append(np.asarray(T, float))
        return len(self.tables) - 1

    def add_table(self, rows, cols, tid, coef):
        n = len(rows)
        self.t_rows.append(np.asarray(rows, np.int64))
        self.t_cols.append(np.asarray(cols, np.int64))
        self.t_tid.append(np.full(n, tid, np.int64))
        self.t_coef.append(np.asarray(coef, float) * np.ones(n))

    def add_dense(self, r, c, block):
        self.d_rows.append(r)
        self.d_cols.append(c)
        self.dense.append(block)

    def finish(self, nblocks, rhs) -> SipTerms:
        N = self.N
        cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)  # noqa: E731
        tr, tc = cat(self.t_rows, np.int64), cat(self.t_cols, np.int64)
        tt, tk = cat(self.t_tid, np.int64), cat(self.t_coef, float)
        dr, dc = np.asarray(self.d_rows, np.int64), np.asarray(self.d_cols, np.int64)
        tkey, dkey = tr * nblocks + tc, dr * nblocks + dc
        keys = np.unique(np.concatenate([tkey, dkey]))
        ot = np.searchsorted(keys, tkey)
        od = np.searchsorted(keys, dkey)
        to = np.argsort(ot, kind="stable")
        do = np.argsort(od, kind="stable")
        nout = len(keys)
        tptr = np.zeros(nout + 1, np.int64)
        np.cumsum(np.bincount(ot, minlength=nout), out=tptr[1:])
        dptr = np.zeros(nout + 1, np.int64)
        np.cumsum(np.bincount(od, minlength=nout), out=dptr[1:])
        rows, cols = keys // nblocks, keys % nblocks
        row_ptr = np.zeros(nblocks + 1, np.int64)
        np.cumsum(np.bincount(rows, minlength=nblocks), out=row_ptr[1:])
        dense = np.stack(self.dense) if self.dense else np.zeros((0, N, N))
        tables = np.stack(self.tables) if self.tables else np.zeros((0, N, N))
        return SipTerms(N, nblocks, row_ptr, cols, tptr, tt[to], tk[to], dptr, do,
                        tables, dense, rhs)


def _ref_cell(cm):
    lo, hi = cm.mesh.bounds(0)
    return np.asarray(lo, float), np.asarray(hi, float)


def sip_terms(cm: CutCellMesh, basis: PlainBasis, problem: PoissonProblem,
              groups, c_eta: float = 4.0, workers: int | None = None) -> SipTerms:
    """Term lists of assemble_sip + assemble_rhs (assembly.py:255-422) with
    the penalty of the small-cell aggregates `groups` (the reference's
    agg_map argument)."""
    if not c_eta > 0:
        raise InvalidConfigError(f"c_eta must be positive, got {c_eta}")
    D, N, k = cm.mesh.dim, basis.size, basis.degree
    mesh, f = cm.mesh, cm.faces
    pidx = PieceIndex.build(cm.species_volume)
    B = pidx.num_blocks
    inv_h = penalty_inv_h(cm, pidx, groups)
    ck2 = c_eta * k * k
    tb = _TermBuilder(N)
    rhs = np.zeros(B * N)
    rlo, rhi = _ref_cell(cm)
    order = cm.gauss_order

    # ---- volume terms ----------------------------------------------------
    rule0 = tensor_rule(rlo, rhi, order)
    V0, G0 = basis.eval_with_grad(rlo, rhi, rule0.nodes)
    tid_K = tb.table(_stiffness(rule0.weights, G0))
    pj, ps = pidx.pieces[:, 0], pidx.pieces[:, 1]
    cut_piece = np.array([(int(a), int(b)) in cm.cut_volume_rules for a, b in pidx.pieces],
                         dtype=bool) if B else np.zeros(0, bool)
    reg = np.flatnonzero(~cut_piece)
    mu_s = np.where(ps == NEG, problem.mu_a, problem.mu_b)
    tb.add_table(reg, reg, tid_K, mu_s[reg])
    # regular rhs: V0^T (w * f(nodes of the cell))
    if len(reg):
        lo_r, hi_r = mesh.bounds(pj[reg])
        ref_nodes = (rule0.nodes - 0.5 * (rhi + rlo)) / (0.5 * (rhi - rlo))
        for c in range(0, len(reg), 65536):
            sl = slice(c, c + 65536)
            nodes = 0.5 * (hi_r[sl] + lo_r[sl])[:, None, :] + ref_nodes[None] * (0.5 * (hi_r[sl] - lo_r[sl]))[:, None, :]
            fv = np.asarray(problem.source(nodes.reshape(-1, D)), float).reshape(len(nodes), -1)
            vec = (fv * rule0.weights[None]) @ V0
            rhs.reshape(B, N)[reg[sl]] += vec
    items = []   # cut items, evaluated in parallel below (reference order kept)
    for b in np.flatnonzero(cut_piece):
        items.append(("vol", int(b), int(pj[b]), int(ps[b])))

    # ---- face tables -------------------------------------------------------
    # reference face of cell 0 along each axis: its hi face (cell 0 = minus
    # side) and the matching lo face of the plus neighbour (shifted cell)
    w = mesh.widths
    face_tabs = {}
    for a in range(D):
        keep = [d for d in range(D) if d != a]
        r = tensor_rule(rlo[keep], rhi[keep], order)
        nodes = embed(r.nodes, a, float(rhi[a]))
        plo, phi_ = rlo.copy(), rhi.copy()
        plo[a] += w[a]
        phi_[a] += w[a]
        Vm, Gm = basis.eval_with_grad(rlo, rhi, nodes)
        Vp, Gp = basis.eval_with_grad(plo, phi_, nodes)
        sides = [(Vm, Gm[:, :, a], 1.0), (Vp, Gp[:, :, a], -1.0)]
        C = _pair_terms(r.weights, 0.0, 0.0, sides)
        P = {(x, y): sx * sy * (sides[x][0] * r.weights[:, None]).T @ sides[y][0]
             for x, (_, _, sx) in enumerate(sides) for y, (_, _, sy) in enumerate(sides)}
        ids = {key: (tb.table(C[key]), tb.table(P[key])) for key in C}
        # boundary: lower side is the cell's lo face (plus cell of the pair)
        bnd = {}
        for side, (V, G, sign) in ((0, (Vp, Gp, -1.0)), (1, (Vm, Gm, 1.0))):
            Cb = _pair_terms(r.weights, 0.0, 0.0, [(V, sign * G[:, :, a], 1.0)])[(0, 0)]
            Pb = (V * r.weights[:, None]).T @ V
            bnd[side] = (tb.table(Cb), tb.table(Pb), V, sign * G[:, :, a], r)
        face_tabs[a] = (ids, bnd)

    # ---- faces ---------------------------------------------------------------
    fsm = cm.face_species_measure
    bmask = f.is_boundary
    stored = np.zeros((len(f), 2), bool)
    for (fid, s) in cm.cut_face_rules:
        stored[fid, s] = True
    for s in SPECIES:
        mu = problem.mu(s)
        # interior faces
        jm, jp = f.minus, f.plus
        ok = (~bmask) & (fsm[:, s] != 0.0)
        ok &= (pidx.block[np.maximum(jm, 0), s] >= 0) & (pidx.block[np.maximum(jp, 0), s] >= 0)
        for a in range(D):
            sel = np.flatnonzero(ok & (f.axis == a) & ~stored[:, s])
            bm, bp = pidx.block[jm[sel], s], pidx.block[jp[sel], s]
            eta = ck2 * np.maximum(inv_h[bm], inv_h[bp])
            ids = face_tabs[a][0]
            for (x, y), (tc, tp) in ids.items():
                rows = bm if x == 0 else bp
                cols = bm if y == 0 else bp
                tb.add_table(rows, cols, tc, mu)
                tb.add_table(rows, cols, tp, eta * mu)
        for fid in np.flatnonzero(ok & stored[:, s]):
            if len(cm.cut_face_rules[(int(fid), s)].weights) == 0:
                continue
            jm_, jp_ = int(jm[fid]), int(jp[fid])
            bm, bp = int(pidx.block[jm_, s]), int(pidx.block[jp_, s])
            eta = ck2 * max(inv_h[bm], inv_h[bp])
            items.append(("face", int(fid), s, int(f.axis[fid]), jm_, jp_, bm, bp, eta, mu))
        # boundary faces
        for a in range(D):
            for side in (0, 1):
                kind, g = problem.condition(a, side)
                cell = f.plus if side == 0 else f.minus
                on = bmask & (f.axis == a) & ((f.minus < 0) if side == 0 else (f.plus < 0))
                on &= (fsm[:, s] != 0.0) & (pidx.block[np.maximum(cell, 0), s] >= 0)
                sign = -1.0 if side == 0 else 1.0
                tc, tp, Vt, Gnt, rt = face_tabs[a][1][side]
                sel = np.flatnonzero(on & ~stored[:, s])
                bb = pidx.block[cell[sel], s]
                eta = ck2 * inv_h[bb]
                if kind != NEUMANN:
                    tb.add_table(bb, bb, tc, mu)
                    tb.add_table(bb, bb, tp, eta * mu)
                if len(sel):
                    # boundary data at every face's own nodes
                    keep = [d for d in range(D) if d != a]
                    ref_nodes = (rt.nodes - 0.5 * (rhi[keep] + rlo[keep])) / (0.5 * (rhi[keep] - rlo[keep]))
                    flo, fhi = f.lo[sel][:, keep], f.hi[sel][:, keep]
                    pts = 0.5 * (fhi + flo)[:, None, :] + ref_nodes[None] * (0.5 * (fhi - flo))[:, None, :]
                    full = np.empty(pts.shape[:2] + (D,))
                    full[..., keep] = pts
                    full[..., a] = f.lo[sel][:, a][:, None]
                    gv = _bvals(g, full.reshape(-1, D), s).reshape(len(sel), -1)
                    if kind == NEUMANN:
                        vec = (gv * (rt.weights * mu)[None]) @ Vt
                    else:
                        vec = np.einsum("fp,fpi->fi", gv * (rt.weights * mu)[None],
                                        eta[:, None, None] * Vt[None] - Gnt[None])
                    np.add.at(rhs.reshape(B, N), bb, vec)
                for fid in np.flatnonzero(on & stored[:, s]):
                    if len(cm.cut_face_rules[(int(fid), s)].weights) == 0:
                        continue
                    j = int(cell[fid])
                    b = int(pidx.block[j, s])
                    items.append(("bface", int(fid), s, a, side, j, b, ck2 * inv_h[b], mu))

    # ---- interface -------------------------------------------------------------
    for j in sorted(cm.interface_rules):
        if len(cm.interface_rules[j].weights) == 0:
            continue
        bn, bp = int(pidx.block[j, NEG]), int(pidx.block[j, POS])
        if bn < 0 or bp < 0:
            raise MissingSpeciesError(f"cell {j}: interface without both species")
        items.append(("iface", int(j), bn, bp, ck2 * max(inv_h[bn], inv_h[bp])))

    for dense, vecs in _eval_items(cm, basis, problem, items, workers):
        for r, c, blk in dense:
            tb.add_dense(r, c, blk)
        for b, vec in vecs:
            rhs[b * N:(b + 1) * N] += vec
    return tb.finish(B, rhs)
