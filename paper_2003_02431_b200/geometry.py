"""Setup row SURVEY 8(f)#1: cut-cell classification and small-cell
agglomeration, matching the reference bit for bit.

The reference (cutcells.py:96-197 -> quadrature.py:444-517) builds full
quadrature rules for every cell; classification (which species are present,
`species_volume > 0`) and agglomeration (fractions, largest neighbour) only
need the *measures* of those rules.  This module reproduces every decision of
the reference's recursive cut-box procedure -- sign probes (Gauss points of
order+2 and corners, ZERO_BAND), the plane-fit linearity test, 2^D
subdivision down to quad_depth, the leaf linearisation, Sutherland-Hodgman
clipping, section polygons, fan triangulation into Duffy triangles /
tetrahedra with the sliver filter -- and forms each rule's weight arrays with
the same floating-point operations, so `species_volume` is the reference's
to the last bit (tests/test_geometry.py pins it against rules the reference
built).  The recursion takes an accumulator: `_Measure` keeps weights only;
cutcells._Rules also forms node coordinates and interface rules (same
operations as the reference's map_triangle / map_tet / tensor_rule), which
the SIP assembly consumes.

Pure cells are classified for the whole mesh at once (vectorised probes);
cells whose probe values come within 1e-9 of zero, and all cut cells, go
through the per-cell restatement.
"""
from __future__ import annotations

import os
from functools import lru_cache

import numpy as np

from .errors import DegenerateLevelSetError, InvalidDomainError, IsolatedSmallCellError

NEG, POS = 0, 1
ZERO_BAND = 1e-12          # quadrature.py:29
LINEAR_REL_TOL = 1e-12     # quadrature.py:30
SLIVER_REL_TOL = 1e-13     # quadrature.py:31
_CHECK_BAND = 1e-9         # vectorised pass hands these cells to the exact path

_EXTRA = {  # asymmetric interior probes of the linearity test (quadrature.py:339-343)
    1: np.array([[0.37], [0.71]]),
    2: np.array([[0.5, 0.5], [0.37, 0.29], [0.71, 0.61]]),
    3: np.array([[0.5, 0.5, 0.5], [0.37, 0.29, 0.43], [0.71, 0.61, 0.83]]),
}


# ---------------------------------------------------------------------------
# level sets (levelset.py:63-126) -- identical arithmetic

class LevelSet:
    """Picklable level-set function (worker processes evaluate it too)."""

    def __init__(self, name: str, params: dict | None = None):
        self.name = name
        p = dict(params or {})
        if name == "sphere":
            self.c = np.asarray(p.get("center", (0.0, 0.0, 0.0)), dtype=float)
            self.r2 = float(p.get("radius", 0.7)) ** 2
        elif name == "plane":
            self.n = np.asarray(p.get("normal", (1.0, 0.0, 0.0)), dtype=float)
            self.off = p.get("offset", 0.0)
        elif name not in ("paper-benchmark", "benchmark"):
            raise ValueError(f"unknown level set name: {name!r}")

    def __call__(self, x):
        if self.name == "sphere":
            d = x - self.c
            return np.einsum("ij,ij->i", d, d) - self.r2
        if self.name == "plane":
            return x @ self.n - self.off
        return x[:, 0] ** 2 + x[:, 1] ** 2 + x[:, 2] ** 3 - 0.49

    def gradient(self, x):
        """Analytic gradients (levelset.py:75-108)."""
        if self.name == "sphere":
            return 2.0 * (x - self.c)
        if self.name == "plane":
            return np.broadcast_to(self.n, x.shape).copy()
        g = np.empty_like(x)
        g[:, 0] = 2 * x[:, 0]
        g[:, 1] = 2 * x[:, 1]
        g[:, 2] = 3 * x[:, 2] ** 2
        return g

    def unit_normal(self, x):
        """grad(phi)/|grad(phi)|, NEG -> POS (levelset.py:52-57)."""
        g = self.gradient(x)
        norms = np.linalg.norm(g, axis=1, keepdims=True)
        norms[norms == 0] = 1.0
        return g / norms


class UnionLevelSet:
    """min of several level sets: NEG inside any of them (e.g. the two
    spheres of BASELINE config 4).  The reference expresses such a field as a
    user LevelSet(phi, grad) (levelset.py:19-35); this is that field."""

    def __init__(self, parts):
        self.parts = list(parts)
        self.name = "union"

    def _vals(self, x):
        return np.stack([p(x) for p in self.parts])

    def __call__(self, x):
        return self._vals(x).min(axis=0)

    def gradient(self, x):
        k = self._vals(x).argmin(axis=0)
        g = np.stack([p.gradient(x) for p in self.parts])
        return g[k, np.arange(len(x))]

    unit_normal = LevelSet.unit_normal


def level_set(name: str, params: dict | None = None) -> LevelSet:
    return LevelSet(name, params)


# ---------------------------------------------------------------------------
# reference rules (weights only)

@lru_cache(maxsize=None)
def _tensor_ref(dim: int, order: int):
    x, w = np.polynomial.legendre.leggauss(order)
    grids = np.meshgrid(*([x] * dim), indexing="ij")
    wgrids = np.meshgrid(*([w] * dim), indexing="ij")
    nodes = np.stack([g.ravel() for g in grids], axis=1)
    weights = np.ones(len(nodes))
    for wg in wgrids:
        weights = weights * wg.ravel()
    return nodes, weights


@lru_cache(maxsize=None)
def _tri_weights(order: int) -> np.ndarray:
    x, w = np.polynomial.legendre.leggauss(order)
    u, wu = 0.5 * (x + 1), 0.5 * w
    U, _ = np.meshgrid(u, u, indexing="ij")
    WU, WV = np.meshgrid(wu, wu, indexing="ij")
    return (WU * WV * (1 - U)).ravel()


@lru_cache(maxsize=None)
def _tet_weights(order: int) -> np.ndarray:
    x, w = np.polynomial.legendre.leggauss(order)
    u, wu = 0.5 * (x + 1), 0.5 * w
    U, V, _ = np.meshgrid(u, u, u, indexing="ij")
    WU, WV, WW = np.meshgrid(wu, wu, wu, indexing="ij")
    return (WU * WV * WW * ((1 - U) ** 2 * (1 - V))).ravel()


@lru_cache(maxsize=None)
def _unit_corners(dim: int) -> np.ndarray:
    return np.array(list(np.ndindex(*([2] * dim))), dtype=float)


def _corners(lo, hi):
    return lo + _unit_corners(len(lo)) * (hi - lo)


def _box_weights(lo, hi, order):
    _, rw = _tensor_ref(len(lo), order)
    return rw * np.prod(0.5 * (hi - lo))


# ---------------------------------------------------------------------------
# per-box machinery

def _probe_class(vals) -> str:
    if np.all(np.abs(vals) < ZERO_BAND):
        return "zero"
    neg, pos = bool(np.any(vals < 0)), bool(np.any(vals > 0))
    if neg and pos:
        return "cut"
    return "neg" if neg else "pos"


def _probes(lo, hi, order):
    ref, _ = _tensor_ref(len(lo), order + 2)
    half, mid = 0.5 * (hi - lo), 0.5 * (hi + lo)
    return np.vstack([mid + ref * half, _corners(lo, hi)])


def _plane_fit(corners, vals):
    A = np.column_stack([np.ones(len(corners)), corners])
    coef, *_ = np.linalg.lstsq(A, vals, rcond=None)
    return coef[0], coef[1:]


def _accept_plane(phi, lo, hi, corners, cvals):
    c0, c = _plane_fit(corners, cvals)
    w = hi - lo
    extra = lo + _EXTRA[len(lo)] * w
    evals = phi(extra)
    scale = max(float(np.max(np.abs(cvals))), float(np.max(np.abs(evals))),
                float(np.abs(c) @ np.abs(w)), 1e-300)
    err = max(float(np.max(np.abs(c0 + corners @ c - cvals))),
              float(np.max(np.abs(c0 + extra @ c - evals))))
    return (c0, c) if err <= LINEAR_REL_TOL * scale else None


def _halfspace_clip(verts, c0, c, keep_neg):
    s = 1.0 if keep_neg else -1.0
    vals = s * (c0 + verts @ c)
    out = []
    m = len(verts)
    for i in range(m):
        va, vb = vals[i], vals[(i + 1) % m]
        a, b = verts[i], verts[(i + 1) % m]
        if va <= 0:
            out.append(a)
        if (va < 0 < vb) or (vb < 0 < va):
            t = va / (va - vb)
            out.append(a + t * (b - a))
    return np.array(out) if out else np.zeros((0, verts.shape[1]))


def _drop_repeats(verts, scale):
    if len(verts) == 0:
        return verts
    kept = []
    for v in verts:
        if not kept or np.linalg.norm(v - kept[-1]) > 1e-12 * scale:
            kept.append(v)
    if len(kept) > 1 and np.linalg.norm(kept[0] - kept[-1]) <= 1e-12 * scale:
        kept.pop()
    return np.array(kept)


def _faces3(lo, hi):
    (x0, y0, z0), (x1, y1, z1) = lo, hi
    return [np.array(f) for f in (
        [[x0, y0, z0], [x0, y1, z0], [x0, y1, z1], [x0, y0, z1]],
        [[x1, y0, z0], [x1, y1, z0], [x1, y1, z1], [x1, y0, z1]],
        [[x0, y0, z0], [x1, y0, z0], [x1, y0, z1], [x0, y0, z1]],
        [[x0, y1, z0], [x1, y1, z0], [x1, y1, z1], [x0, y1, z1]],
        [[x0, y0, z0], [x1, y0, z0], [x1, y1, z0], [x0, y1, z0]],
        [[x0, y0, z1], [x1, y0, z1], [x1, y1, z1], [x0, y1, z1]])]


def _section(lo, hi, c0, c):
    corners = _corners(lo, hi)
    vals = c0 + corners @ c
    pts = []
    for i in range(8):
        for j in range(i + 1, 8):
            if (corners[i] != corners[j]).sum() != 1:
                continue
            va, vb = vals[i], vals[j]
            if (va < 0 < vb) or (vb < 0 < va):
                t = va / (va - vb)
                pts.append(corners[i] + t * (corners[j] - corners[i]))
    if len(pts) < 3:
        return np.zeros((0, 3))
    pts = np.array(pts)
    ctr = pts.mean(axis=0)
    n = c / np.linalg.norm(c)
    u = np.cross(n, np.eye(3)[np.argmin(np.abs(n))])
    u /= np.linalg.norm(u)
    v = np.cross(n, u)
    order = np.argsort(np.arctan2((pts - ctr) @ v, (pts - ctr) @ u))
    return _drop_repeats(pts[order], float(np.linalg.norm(hi - lo)))


class _Measure:
    """Weight arrays per species in the reference's accumulation order.  The
    `nodes` callables are only invoked by accumulators that keep nodes
    (cutcells._Rules); measures never build coordinates."""

    want_interface = False

    def __init__(self):
        self.w = {NEG: [], POS: []}

    def add(self, s, weights, nodes=None):
        if len(weights):
            self.w[s].append(weights)

    def add_interface(self, weights, nodes):
        pass

    def measure(self, s) -> float:
        if not self.w[s]:
            return 0.0
        return float(np.concatenate(self.w[s]).sum())


@lru_cache(maxsize=None)
def _tri_nodes(order: int) -> np.ndarray:
    """Duffy nodes of the unit triangle (quadrature.py:93-103)."""
    x, _ = np.polynomial.legendre.leggauss(order)
    u = 0.5 * (x + 1)
    U, V = np.meshgrid(u, u, indexing="ij")
    return np.stack([U.ravel(), (V * (1 - U)).ravel()], axis=1)


@lru_cache(maxsize=None)
def _tet_nodes(order: int) -> np.ndarray:
    """Duffy nodes of the unit tetrahedron (quadrature.py:106-121)."""
    x, _ = np.polynomial.legendre.leggauss(order)
    u = 0.5 * (x + 1)
    U, V, W = np.meshgrid(u, u, u, indexing="ij")
    return np.stack([U.ravel(), (V * (1 - U)).ravel(), (W * (1 - U) * (1 - V)).ravel()], axis=1)


def _box_nodes(lo, hi, order):
    ref, _ = _tensor_ref(len(lo), order)
    return 0.5 * (hi + lo) + ref * (0.5 * (hi - lo))


def _tri_map(p0, e1, e2, order):
    r = _tri_nodes(order)
    return p0 + np.outer(r[:, 0], e1) + np.outer(r[:, 1], e2)


def _clip_leaf(lo, hi, c0, c, order, acc):
    """Exact rules of a box cut by the plane c0 + c.x = 0
    (_clip_box_rules, quadrature.py:366-437)."""
    dim = len(lo)
    if float(np.linalg.norm(c)) < 1e-300:
        acc.add(NEG if c0 < 0 else POS, _box_weights(lo, hi, order),
                lambda: _box_nodes(lo, hi, order))
        return
    if dim == 1:
        root = min(max(-c0 / c[0], lo[0]), hi[0])
        lo_s = NEG if c[0] > 0 else POS
        for s, (a, b) in ((lo_s, (lo[0], root)), (1 - lo_s, (root, hi[0]))):
            if b - a > SLIVER_REL_TOL * (hi[0] - lo[0]):
                al, bl = np.array([a]), np.array([b])
                acc.add(s, _box_weights(al, bl, order),
                        lambda al=al, bl=bl: _box_nodes(al, bl, order))
        return
    if dim == 2:
        ring = np.array([[lo[0], lo[1]], [hi[0], lo[1]], [hi[0], hi[1]], [lo[0], hi[1]]])
        area = float(np.prod(hi - lo))
        tw = _tri_weights(order)
        for s, keep in ((NEG, True), (POS, False)):
            poly = _drop_repeats(_halfspace_clip(ring, c0, c, keep),
                                 float(np.linalg.norm(hi - lo)))
            for i in range(1, len(poly) - 1) if len(poly) >= 3 else ():
                e1, e2 = poly[i] - poly[0], poly[i + 1] - poly[0]
                wts = tw * abs(e1[0] * e2[1] - e1[1] * e2[0])
                if wts.sum() > SLIVER_REL_TOL * area:
                    acc.add(s, wts, lambda p0=poly[0], e1=e1, e2=e2: _tri_map(p0, e1, e2, order))
        if acc.want_interface:
            vals = c0 + ring @ c
            pts = []
            for i in range(4):
                va, vb = vals[i], vals[(i + 1) % 4]
                a, b = ring[i], ring[(i + 1) % 4]
                if (va < 0 < vb) or (vb < 0 < va):
                    t = va / (va - vb)
                    pts.append(a + t * (b - a))
            if len(pts) >= 2:
                pts = np.array(pts)
                proj = pts @ np.array([-c[1], c[0]])
                p0, p1 = pts[np.argmin(proj)], pts[np.argmax(proj)]
                length = float(np.linalg.norm(p1 - p0))
                if length > SLIVER_REL_TOL * float(np.linalg.norm(hi - lo)):
                    x1, w1 = np.polynomial.legendre.leggauss(order)
                    acc.add_interface(0.5 * w1 * length,
                                      lambda: p0 + np.outer(0.5 * (x1 + 1), p1 - p0))
        return
    vol = float(np.prod(hi - lo))
    diam = float(np.linalg.norm(hi - lo))
    sec = _section(lo, hi, c0, c)
    tw = _tet_weights(order)
    for s, keep in ((NEG, True), (POS, False)):
        polys = [_drop_repeats(_halfspace_clip(f, c0, c, keep), diam) for f in _faces3(lo, hi)]
        if len(sec) >= 3:
            polys.append(sec)
        verts = [p for poly in polys if len(poly) >= 3 for p in poly]
        if not verts:
            continue
        apex = np.mean(verts, axis=0)
        for poly in polys:
            if len(poly) < 3:
                continue
            for i in range(1, len(poly) - 1):
                B = np.stack([poly[0] - apex, poly[i] - apex, poly[i + 1] - apex], axis=1)
                wts = tw * abs(np.linalg.det(B))
                if wts.sum() > SLIVER_REL_TOL * vol:
                    acc.add(s, wts, lambda B=B, apex=apex: apex + _tet_nodes(order) @ B.T)
    if acc.want_interface and len(sec) >= 3:
        tw2 = _tri_weights(order)
        for i in range(1, len(sec) - 1):
            e1, e2 = sec[i] - sec[0], sec[i + 1] - sec[0]
            wts = tw2 * float(np.linalg.norm(np.cross(e1, e2)))
            if wts.sum() > SLIVER_REL_TOL * diam ** 2:
                acc.add_interface(wts, lambda p0=sec[0], e1=e1, e2=e2: _tri_map(p0, e1, e2, order))


def _recurse(phi, lo, hi, depth, order, leaf_order, acc):
    cls = _probe_class(phi(_probes(lo, hi, order)))
    if cls == "zero":
        return
    if cls in ("neg", "pos"):
        acc.add(NEG if cls == "neg" else POS, _box_weights(lo, hi, order),
                lambda: _box_nodes(lo, hi, order))
        return
    corners = _corners(lo, hi)
    cvals = phi(corners)
    plane = _accept_plane(phi, lo, hi, corners, cvals)
    if plane is not None:
        _clip_leaf(lo, hi, plane[0], plane[1], order, acc)
        return
    if depth > 0:
        mid = 0.5 * (lo + hi)
        for bits in np.ndindex(*([2] * len(lo))):
            b = np.array(bits)
            _recurse(phi, np.where(b == 0, lo, mid), np.where(b == 0, mid, hi),
                     depth - 1, order, leaf_order, acc)
        return
    c0, c = _plane_fit(corners, cvals)
    _clip_leaf(lo, hi, c0, c, leaf_order, acc)


def cell_species_volumes(phi, lo, hi, depth: int, order: int, leaf_order: int = 2):
    """(vol_NEG, vol_POS) of one box: the measures of cut_box_rules
    (quadrature.py:478-517)."""
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    if _probe_class(phi(_probes(lo, hi, order))) == "zero":
        raise DegenerateLevelSetError(f"level set vanishes on the whole box {lo} .. {hi}")
    acc = _Measure()
    _recurse(phi, lo, hi, depth, order, leaf_order, acc)
    return acc.measure(NEG), acc.measure(POS)


# ---------------------------------------------------------------------------
# whole mesh

class CartesianMesh:
    """Axis-aligned Cartesian mesh, x fastest (mesh.py:19-68, 130-159)."""

    def __init__(self, box, cells_per_axis):
        self.dim = len(box)
        if self.dim not in (2, 3) or len(cells_per_axis) != self.dim:
            raise InvalidDomainError("dimension must be 2 or 3")
        self.box = tuple((float(a), float(b)) for a, b in box)
        self.n = tuple(int(c) for c in cells_per_axis)
        self.widths = np.array([(b - a) / c for (a, b), c in zip(self.box, self.n)])
        self.num_cells = int(np.prod(self.n))
        self.cell_volume = float(np.prod(self.widths))

    def multi(self, j):
        out = []
        for c in self.n:
            out.append(j % c)
            j = j // c
        return np.stack(out, axis=-1)

    def bounds(self, j):
        m = self.multi(np.asarray(j))
        lo = np.stack([self.box[a][0] + m[..., a] * self.widths[a]
                       for a in range(self.dim)], axis=-1)
        return lo, lo + self.widths

    def adjacency(self):
        """Sorted face neighbours of every cell (mesh.py:200-215)."""
        J = self.num_cells
        m = self.multi(np.arange(J))
        strides = np.cumprod((1,) + self.n[:-1])
        nbrs = [[] for _ in range(J)]
        for a in range(self.dim):
            ok = m[:, a] + 1 < self.n[a]
            src = np.flatnonzero(ok)
            dst = src + strides[a]
            for s_, d_ in zip(src, dst):
                nbrs[s_].append(int(d_))
                nbrs[d_].append(int(s_))
        return [sorted(x) for x in nbrs]


def _cells_job(args):
    phi, los, his, depth, order, cells = args
    vols = np.zeros((len(cells), 2))
    for i, j in enumerate(cells):
        try:
            vols[i] = cell_species_volumes(phi, los[i], his[i], depth, order)
        except DegenerateLevelSetError as exc:
            raise DegenerateLevelSetError(f"cell {j}: {exc}") from exc
    return cells, vols


def species_volumes(mesh: CartesianMesh, phi, quad_depth: int, gauss_order: int,
                    workers: int | None = None):
    """species_volume (num_cells, 2) of classify_and_build (cutcells.py:105-127).
    Cut cells are spread over `workers` processes (default: all cores when
    there are >= 64 of them); the result does not depend on the split."""
    J, dim = mesh.num_cells, mesh.dim
    lo, hi = mesh.bounds(np.arange(J))
    ref, _ = _tensor_ref(dim, gauss_order + 2)
    half, mid = 0.5 * (hi - lo), 0.5 * (hi + lo)
    probes = mid[:, None, :] + ref[None, :, :] * half[:, None, :]
    corners = lo[:, None, :] + _unit_corners(dim)[None, :, :] * (hi - lo)[:, None, :]
    pts = np.concatenate([probes, corners], axis=1)
    P = pts.shape[1]
    vals = phi(pts.reshape(-1, dim)).reshape(J, P)
    neg, pos = (vals < 0).any(1), (vals > 0).any(1)
    exact = (neg & pos) | (np.abs(vals).min(1) < _CHECK_BAND)
    out = np.zeros((J, 2))
    # pure cells: the tensor-rule measure of their own box
    _, rw = _tensor_ref(dim, gauss_order)
    pvol = np.prod(half, axis=1)
    cache: dict = {}
    pure = np.flatnonzero(~exact)
    for j in pure:
        p = pvol[j]
        m = cache.get(p)
        if m is None:
            m = float((rw * p).sum())
            cache[p] = m
        out[j, NEG if neg[j] else POS] = m
    todo = np.flatnonzero(exact)
    if workers is None:
        workers = min(os.cpu_count() or 1, 16) if len(todo) >= 64 else 1
    if workers > 1 and len(todo) > 1:
        from concurrent.futures import ProcessPoolExecutor

        chunks = np.array_split(todo, workers * 4)
        jobs = [(phi, lo[c], hi[c], quad_depth, gauss_order, c) for c in chunks if len(c)]
        with ProcessPoolExecutor(max_workers=workers) as pool:
            for cells, vols in pool.map(_cells_job, jobs):
                out[cells] = vols
    else:
        _, vols = _cells_job((phi, lo[todo], hi[todo], quad_depth, gauss_order, todo))
        out[todo] = vols
    return out


def small_cell_pairs(species_volume, cell_volume, adjacency, alpha: float):
    """Edges of small_cell_agglomeration_map (agglomeration.py:41-76): every
    present piece with fraction in (0, alpha] merges into its largest
    same-species face neighbour (ties: smaller cell index)."""
    if not 0 <= alpha < 1:
        raise ValueError(f"alpha must be in [0, 1), got {alpha}")
    edges = set()
    if alpha == 0:
        return edges
    J = len(species_volume)
    for j in range(J):
        for s in (NEG, POS):
            v = species_volume[j, s]
            if not v > 0:
                continue
            frac = float(v / cell_volume)
            if not 0 < frac <= alpha:
                continue
            cand = [l for l in adjacency[j] if species_volume[l, s] > 0]
            if not cand:
                raise IsolatedSmallCellError(
                    f"cell {j} species {s} (fraction {frac:.4g}) has no same-species "
                    "face neighbor")
            best = min(cand, key=lambda l: (-species_volume[l, s], l))
            edges.add(tuple(sorted(((j, s), (best, s)))))
    return edges


def aggregates(species_volume, edges):
    """Connected components over present pieces (cut_aggregates,
    agglomeration.py:102-123): sorted by minimum piece, members sorted."""
    pieces = [(j, s) for j in range(len(species_volume)) for s in (NEG, POS)
              if species_volume[j, s] > 0]
    index = {p: i for i, p in enumerate(pieces)}
    parent = list(range(len(pieces)))

    def root(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x

    for a, b in sorted(edges):
        ra, rb = root(index[a]), root(index[b])
        if ra != rb:
            ra, rb = min(ra, rb), max(ra, rb)
            parent[rb] = ra
    groups: dict = {}
    for p, i in index.items():
        groups.setdefault(root(i), []).append(p)
    return [sorted(groups[r]) for r in sorted(groups)]


def axis_block_edges(mesh: CartesianMesh, level: int):
    """Mesh-graph edges (a < b) inside the same axis-aligned index block of
    width 2^(level-1), the last block per axis absorbing the remainder
    (build_multigrid_aggregation_sequence, mesh.py:254-287)."""
    width = 2 ** (level - 1)
    J = mesh.num_cells
    m = mesh.multi(np.arange(J))
    nblocks = np.maximum(np.array(mesh.n) // width, 1)
    blk = np.minimum(m // width, nblocks - 1)
    strides = np.cumprod((1,) + mesh.n[:-1])
    out = []
    for a in range(mesh.dim):
        src = np.flatnonzero(m[:, a] + 1 < mesh.n[a])
        dst = src + strides[a]
        same = np.all(blk[src] == blk[dst], axis=1)
        out += list(zip(src[same].tolist(), dst[same].tolist()))
    return out


def lift_edges(bg_edges, species_volume):
    """Background edges duplicated per species present on both cells
    (lift_aggregation_to_cutcells, agglomeration.py:79-93)."""
    edges = set()
    for a, b in bg_edges:
        for s in (NEG, POS):
            if species_volume[a, s] > 0 and species_volume[b, s] > 0:
                edges.add(tuple(sorted(((a, s), (b, s)))))
    return edges


def level_aggregates(mesh: CartesianMesh, species_volume, small_edges, num_levels: int):
    """Aggregates of hierarchy levels 1..num_levels (build_hierarchy,
    transfer.py:480-500): level 1 = small-cell map; level l = lifted axis
    blocks of width 2^(l-1) united with the small-cell map."""
    out = [aggregates(species_volume, small_edges)]
    for lam in range(2, num_levels + 1):
        eff = lift_edges(axis_block_edges(mesh, lam), species_volume) | set(small_edges)
        out.append(aggregates(species_volume, eff))
    return out
