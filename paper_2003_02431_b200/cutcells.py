"""Cut-cell meshes with full quadrature rules (SURVEY 8(f)#2 input).

Restates classify_and_build (cutcells.py:96-197 of the reference) on top of
the bit-exact cut-box recursion in geometry.py: per cut cell the species
volume rules and the interface rule with unit normals, per face touching a
cut (or mixed) cell the species face rules.  Pure cells and full faces keep
no stored rule; `quad_volume` / `quad_cut_face` build their tensor rules on
demand exactly as the reference does (cutcells.py:211-250).

Layout: faces are arrays (axis, minus, plus, lo, hi) in the reference's
enumeration order (mesh.py:155-197, axis-major, then plane, then the cross
section with the last axis fastest); -1 marks a missing neighbour.  Cut cells
and cut faces are processed in worker processes; results do not depend on
the split.
"""
from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from .errors import DegenerateLevelSetError, MissingSpeciesError
from .geometry import (
    NEG,
    POS,
    _CHECK_BAND,
    CartesianMesh,
    _box_nodes,
    _box_weights,
    _Measure,
    _probe_class,
    _probes,
    _recurse,
    _tensor_ref,
    _unit_corners,
)

SPECIES = (NEG, POS)
PURE_NEG, PURE_POS, CUT = 0, 1, 2


@dataclass
class QuadRule:
    nodes: np.ndarray
    weights: np.ndarray
    normals: np.ndarray | None = None

    @property
    def measure(self) -> float:
        return float(self.weights.sum()) if len(self.weights) else 0.0


class _Rules(_Measure):
    """Accumulator keeping nodes and the interface rule (_Accumulator,
    quadrature.py:290-327)."""

    def __init__(self, dim: int, want_interface: bool):
        super().__init__()
        self.dim = dim
        self.want_interface = want_interface
        self.n = {NEG: [], POS: []}
        self.iw, self.iN = [], []

    def add(self, s, weights, nodes=None):
        if len(weights):
            self.w[s].append(weights)
            self.n[s].append(nodes())

    def add_interface(self, weights, nodes):
        if self.want_interface and len(weights):
            self.iw.append(weights)
            self.iN.append(nodes())

    def rule(self, s) -> QuadRule:
        if not self.w[s]:
            return QuadRule(np.zeros((0, self.dim)), np.zeros(0))
        return QuadRule(np.concatenate(self.n[s]), np.concatenate(self.w[s]))

    def interface(self) -> QuadRule:
        if not self.iw:
            return QuadRule(np.zeros((0, self.dim)), np.zeros(0))
        return QuadRule(np.concatenate(self.iN), np.concatenate(self.iw))


def cut_box_rules(phi, lo, hi, depth, order, want_interface=False, leaf_order=2,
                  on_degenerate="raise"):
    """Both species' volume rules (+ interface) of a box (quadrature.py:478-517)."""
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    if _probe_class(phi(_probes(lo, hi, order))) == "zero":
        if on_degenerate == "raise":
            raise DegenerateLevelSetError(f"level set vanishes on the whole box {lo} .. {hi}")
        e = QuadRule(np.zeros((0, len(lo))), np.zeros(0))
        return {NEG: e, POS: e, "interface": e}
    acc = _Rules(len(lo), want_interface)
    _recurse(phi, lo, hi, depth, order, leaf_order, acc)
    return {NEG: acc.rule(NEG), POS: acc.rule(POS), "interface": acc.interface()}


def tensor_rule(lo, hi, order) -> QuadRule:
    lo = np.asarray(lo, float)
    hi = np.asarray(hi, float)
    return QuadRule(_box_nodes(lo, hi, order), _box_weights(lo, hi, order).copy())


def embed(points, axis, coord):
    n, dm1 = points.shape
    out = np.empty((n, dm1 + 1))
    out[:, :axis] = points[:, :axis]
    out[:, axis] = coord
    out[:, axis + 1:] = points[:, axis:]
    return out


class _FacePhi:
    def __init__(self, phi, axis, coord):
        self.phi, self.axis, self.coord = phi, axis, coord

    def __call__(self, pts):
        return self.phi(embed(pts, self.axis, self.coord))


# ---------------------------------------------------------------------------
# faces

@dataclass
class Faces:
    axis: np.ndarray    # (F,) int
    minus: np.ndarray   # (F,) int, -1 = boundary
    plus: np.ndarray    # (F,) int, -1 = boundary
    lo: np.ndarray      # (F, D)
    hi: np.ndarray      # (F, D)

    def __len__(self):
        return len(self.axis)

    @property
    def is_boundary(self):
        return (self.minus < 0) | (self.plus < 0)

    def area(self) -> np.ndarray:
        """_face_area (cutcells.py:200-205): product over the in-face axes."""
        a = np.ones(len(self))
        for d in range(self.lo.shape[1]):
            on = self.axis != d
            a = np.where(on, a * (self.hi[:, d] - self.lo[:, d]), a)
        return a

    def box(self, f):
        """The face as a (D-1)-box: (lo, hi, axis, coordinate)."""
        ax = int(self.axis[f])
        keep = [d for d in range(self.lo.shape[1]) if d != ax]
        return self.lo[f, keep], self.hi[f, keep], ax, float(self.lo[f, ax])


def enumerate_faces(mesh: CartesianMesh) -> Faces:
    """All faces in the reference order (mesh.py:155-197)."""
    D, n, w = mesh.dim, mesh.n, mesh.widths
    strides = np.cumprod((1,) + n[:-1])
    parts = []
    for axis in range(D):
        other = [a for a in range(D) if a != axis]
        shape = (n[axis] + 1,) + tuple(n[a] for a in other)
        idx = np.indices(shape).reshape(len(shape), -1)
        plane = idx[0]
        multi = np.zeros((D, idx.shape[1]), np.int64)
        for k, a in enumerate(other):
            multi[a] = idx[k + 1]
        base = sum(multi[a] * strides[a] for a in other)
        minus = np.where(plane > 0, base + (plane - 1) * strides[axis], -1)
        plus = np.where(plane < n[axis], base + plane * strides[axis], -1)
        lo = np.empty((idx.shape[1], D))
        hi = np.empty((idx.shape[1], D))
        for a in range(D):
            if a == axis:
                lo[:, a] = hi[:, a] = mesh.box[a][0] + plane * w[a]
            else:
                lo[:, a] = mesh.box[a][0] + multi[a] * w[a]
                hi[:, a] = lo[:, a] + w[a]
        parts.append((np.full(idx.shape[1], axis), minus, plus, lo, hi))
    cat = [np.concatenate([p[i] for p in parts]) for i in range(5)]
    return Faces(*cat)


# ---------------------------------------------------------------------------
# mesh

@dataclass
class CutCellMesh:
    mesh: CartesianMesh
    level_set: object
    quad_depth: int
    gauss_order: int
    species_volume: np.ndarray     # (J, 2)
    faces: Faces
    face_species_measure: np.ndarray  # (F, 2)
    cut_volume_rules: dict         # (cell, species) -> QuadRule
    interface_rules: dict          # cell -> QuadRule with normals
    cut_face_rules: dict           # (face, species) -> QuadRule

    @property
    def num_cells(self):
        return self.mesh.num_cells

    def present(self, j, s):
        return self.species_volume[j, s] > 0.0

    def is_cut(self, j):
        return self.present(j, NEG) and self.present(j, POS)

    def interface_measure(self, j) -> float:
        r = self.interface_rules.get(j)
        return r.measure if r is not None else 0.0

    def interface_measures(self) -> np.ndarray:
        out = np.zeros(self.num_cells)
        for j, r in self.interface_rules.items():
            out[j] = r.measure
        return out


def quad_volume(cm: CutCellMesh, j, s) -> QuadRule:
    if not cm.present(j, s):
        raise MissingSpeciesError(f"species {s} absent in cell {j}")
    r = cm.cut_volume_rules.get((j, s))
    if r is not None:
        return r
    lo, hi = cm.mesh.bounds(j)
    return tensor_rule(lo, hi, cm.gauss_order)


def quad_cut_face(cm: CutCellMesh, f, s) -> QuadRule:
    cells = [c for c in (cm.faces.minus[f], cm.faces.plus[f]) if c >= 0]
    if not any(cm.present(c, s) for c in cells):
        raise MissingSpeciesError(f"species {s} absent on both sides of face {f}")
    r = cm.cut_face_rules.get((f, s))
    if r is not None:
        return r
    D = cm.mesh.dim
    if cm.face_species_measure[f, s] == 0.0:
        return QuadRule(np.zeros((0, D)), np.zeros(0))
    flo, fhi, ax, coord = cm.faces.box(f)
    r = tensor_rule(flo, fhi, cm.gauss_order)
    return QuadRule(embed(r.nodes, ax, coord), r.weights)


def _nontrivial(rule: QuadRule, lo, hi) -> bool:
    vol = float(np.prod(hi - lo))
    return abs(rule.measure - vol) > 1e-10 * vol


def _cell_job(args):
    phi, los, his, depth, order, cells = args
    out = []
    for i, j in enumerate(cells):
        lo, hi = los[i], his[i]
        try:
            rules = cut_box_rules(phi, lo, hi, depth, order, want_interface=True)
        except DegenerateLevelSetError as exc:
            raise DegenerateLevelSetError(f"cell {j}: {exc}") from exc
        vol = (rules[NEG].measure, rules[POS].measure)
        keep = {s: rules[s] for s in SPECIES if vol[s] > 0 and _nontrivial(rules[s], lo, hi)}
        iface = rules["interface"]
        if vol[NEG] > 0 and vol[POS] > 0 and len(iface.weights) > 0:
            iface.normals = phi.unit_normal(iface.nodes)
        else:
            iface = None
        out.append((int(j), vol, keep, iface))
    return out


def _face_job(args):
    phi, items, depth, order = args
    out = []
    for f, flo, fhi, ax, coord in items:
        rules = cut_box_rules(_FacePhi(phi, ax, coord), flo, fhi, depth, order,
                              want_interface=False, on_degenerate="empty")
        res = {}
        for s in SPECIES:
            r = rules[s]
            res[s] = (r.measure, QuadRule(embed(r.nodes, ax, coord), r.weights)
                      if len(r.weights) else None)
        out.append((f, res))
    return out


def _run(fn, jobs, workers):
    if workers > 1 and len(jobs) > 1:
        from concurrent.futures import ProcessPoolExecutor

        from ._pool import _init_worker

        with ProcessPoolExecutor(max_workers=workers, initializer=_init_worker) as pool:
            for res in pool.map(fn, jobs):
                yield from res
    else:
        for job in jobs:
            yield from fn(job)


def classify_and_build(mesh: CartesianMesh, level_set, quad_depth: int = 2,
                       gauss_order: int = 4, workers: int | None = None) -> CutCellMesh:
    """classify_and_build (cutcells.py:96-197): species volumes, stored cut
    rules (volume, interface with normals, faces).  Pure cells are found by a
    whole-mesh vectorised probe pass; every cell whose probes come within
    1e-9 of zero goes through the exact per-cell restatement."""
    J, D = mesh.num_cells, mesh.dim
    lo, hi = mesh.bounds(np.arange(J))
    ref, _ = _tensor_ref(D, gauss_order + 2)
    half, mid = 0.5 * (hi - lo), 0.5 * (hi + lo)
    pts = np.concatenate([mid[:, None, :] + ref[None] * half[:, None, :],
                          lo[:, None, :] + _unit_corners(D)[None] * (hi - lo)[:, None, :]], axis=1)
    vals = level_set(pts.reshape(-1, D)).reshape(J, -1)
    neg, pos = (vals < 0).any(1), (vals > 0).any(1)
    exact = (neg & pos) | (np.abs(vals).min(1) < _CHECK_BAND)
    species_volume = np.zeros((J, 2))
    _, rw = _tensor_ref(D, gauss_order)
    pvol = np.prod(half, axis=1)
    cache: dict = {}
    for j in np.flatnonzero(~exact):
        p = pvol[j]
        m = cache.get(p)
        if m is None:
            m = cache[p] = float((rw * p).sum())
        species_volume[j, NEG if neg[j] else POS] = m
    if workers is None:
        workers = min(os.cpu_count() or 1, 16)
    todo = np.flatnonzero(exact)
    nchunks = max(1, min(len(todo), workers * 4))
    jobs = [(level_set, lo[c], hi[c], quad_depth, gauss_order, c)
            for c in np.array_split(todo, nchunks) if len(c)]
    cut_volume_rules, interface_rules = {}, {}
    for j, vol, keep, iface in _run(_cell_job, jobs, workers if len(todo) >= 32 else 1):
        species_volume[j] = vol
        for s, r in keep.items():
            cut_volume_rules[(j, s)] = r
        if iface is not None:
            interface_rules[j] = iface

    faces = enumerate_faces(mesh)
    F = len(faces)
    cls = np.where((species_volume[:, NEG] > 0) & (species_volume[:, POS] > 0), CUT,
                   np.where(species_volume[:, NEG] > 0, PURE_NEG, PURE_POS))
    cm_ = np.where(faces.minus >= 0, cls[np.maximum(faces.minus, 0)], -1)
    cp_ = np.where(faces.plus >= 0, cls[np.maximum(faces.plus, 0)], -1)
    all_neg = ((cm_ == PURE_NEG) | (cm_ < 0)) & ((cp_ == PURE_NEG) | (cp_ < 0))
    all_pos = ((cm_ == PURE_POS) | (cm_ < 0)) & ((cp_ == PURE_POS) | (cp_ < 0))
    fsm = np.zeros((F, 2))
    area = faces.area()
    fsm[all_neg, NEG] = area[all_neg]
    fsm[all_pos, POS] = area[all_pos]
    cutf = np.flatnonzero(~(all_neg | all_pos))
    items = [(int(f),) + faces.box(f) for f in cutf]
    nchunks = max(1, min(len(items), workers * 4))
    fjobs = [(level_set, [items[i] for i in c], quad_depth, gauss_order)
             for c in np.array_split(np.arange(len(items)), nchunks) if len(c)]
    cut_face_rules = {}
    for f, res in _run(_face_job, fjobs, workers if len(items) >= 64 else 1):
        for s in SPECIES:
            fsm[f, s] = res[s][0]
            if res[s][1] is not None:
                cut_face_rules[(f, s)] = res[s][1]
    return CutCellMesh(mesh, level_set, quad_depth, gauss_order, species_volume, faces,
                       fsm, cut_volume_rules, interface_rules, cut_face_rules)
