"""Setup row SURVEY 8(f)#2 on the host: cut-cell quadrature rules bit-exact
against the reference's (digests in setup_<case>.npz), the raw SIP system
(assembly.py:255-422) and the aggregation hierarchy (transfer.py:107-522)
against the reference's level operators (<case>.npz).

The raw operator's product path is the xdg_assemble_blocks kernel
(test_setup_gpu.py); here the same term lists are evaluated on the host
(SipTerms.evaluate_host, test infrastructure) and the Galerkin products are a
host restatement of the kernel's association.
"""
import hashlib
import json

import numpy as np
import pytest

from paper_2003_02431_b200.assembly import PieceIndex, PlainBasis, dirichlet_problem, sip_terms
from paper_2003_02431_b200.case import BenchCase, make_level_set
from paper_2003_02431_b200.cutcells import classify_and_build
from paper_2003_02431_b200.geometry import CartesianMesh, level_aggregates, small_cell_pairs
from paper_2003_02431_b200.hierarchy import fixture_array
from paper_2003_02431_b200.transfer import (
    LevelBuilder,
    aggregate_graph,
    aggregation_level_data,
    build_restriction,
    galerkin_symbolic,
    initial_restriction,
    restrict_rhs,
)

from conftest import golden_path

CASES = ["bench4", "cfg1"]
# level-operator tolerance (max |dM| / max |M|): the reference reproduces its
# own fixtures only to ~1e-10 at p=3 (BLAS-order spread); p=2 cases
# agree to ~1e-13.
TOL = {"bench4": 1e-12, "cfg1": 1e-12}


def _digest(rule):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(rule.nodes, np.float64).tobytes())
    h.update(np.ascontiguousarray(rule.weights, np.float64).tobytes())
    if rule.normals is not None:
        h.update(np.ascontiguousarray(rule.normals, np.float64).tobytes())
    return h.hexdigest()


def case_of(name):
    z = np.load(golden_path(name))
    meta = json.loads(bytes(z["meta"]).decode())
    lp = {k: tuple(v) if isinstance(v, list) else v for k, v in meta["levelset_params"].items()}
    return BenchCase(dim=meta["dim"], cells=meta["cells"], degree=meta["degree"],
                     levelset=meta["levelset"], levelset_params=lp,
                     num_levels=meta["num_levels"]), z


_CACHE = {}


def host_setup(name):
    if name in _CACHE:
        return _CACHE[name]
    c, z = case_of(name)
    mesh = CartesianMesh([(-1.0, 1.0)] * c.dim, [c.cells] * c.dim)
    cm = classify_and_build(mesh, make_level_set(c.levelset, c.levelset_params),
                            c.quad_depth, c.resolved_gauss_order, workers=1)
    small = small_cell_pairs(cm.species_volume, mesh.cell_volume, mesh.adjacency(),
                             c.resolved_alpha)
    groups = level_aggregates(mesh, cm.species_volume, small, c.num_levels)
    basis = PlainBasis(c.degree, c.dim)
    terms = sip_terms(cm, basis, dirichlet_problem(c.mu_a, c.mu_b, dim=c.dim), groups[0])
    _CACHE[name] = (c, z, mesh, cm, groups, basis, terms)
    return _CACHE[name]


def host_galerkin(rp, col, val, R):
    """R^T M R with the kernel's association: per output block, per fine row
    i, P_i = sum_k M_ik R_k, then acc += R_i^T P_i."""
    Rrp, Rcol, Rval = R
    n = int(Rcol.max()) + 1
    crp, ccol, tptr, te, tri, trk = galerkin_symbolic(rp, col, Rrp, Rcol, n)
    out = np.zeros((len(ccol),) + val.shape[1:])
    for o in range(len(ccol)):
        acc, P = 0.0, 0.0
        for t in range(tptr[o], tptr[o + 1]):
            P = P + val[te[t]] @ Rval[trk[t]]
            if t + 1 == tptr[o + 1] or tri[t + 1] != tri[t]:
                acc = acc + Rval[tri[t]].T @ P
                P = 0.0
        out[o] = acc
    return crp, ccol, out


@pytest.mark.parametrize("name", CASES)
def test_rules_bit_exact(name):
    _, _, _, cm, _, _, _ = host_setup(name)
    g = np.load(golden_path(f"setup_{name}"))
    assert np.array_equal(cm.species_volume, g["species_volume"])
    assert np.array_equal(cm.face_species_measure, g["face_species_measure"])
    for label, rules, key in (("vol", cm.cut_volume_rules, lambda k: (k[0], k[1])),
                              ("iface", cm.interface_rules, lambda k: (k, -1)),
                              ("face", cm.cut_face_rules, lambda k: (k[0], k[1]))):
        keys = sorted(rules)
        assert [key(k) for k in keys] == [tuple(r) for r in g[f"{label}_keys"].tolist()], label
        npts = [len(rules[k].weights) for k in keys]
        assert npts == g[f"{label}_npts"].tolist(), label
        sha = [_digest(rules[k]) for k in keys]
        bad = [k for k, a, b in zip(keys, sha, g[f"{label}_sha"].tolist()) if a != b]
        assert not bad, f"{label} rules differ from the reference at {bad[:5]}"


@pytest.mark.parametrize("name", CASES)
def test_raw_system(name):
    _, _, _, _, _, _, T = host_setup(name)
    g = np.load(golden_path(f"setup_{name}"))
    assert np.array_equal(T.row_ptr, g["raw_row_ptr"])
    assert np.array_equal(T.col, g["raw_col"])
    ref = g["raw_val"]
    err = np.abs(T.evaluate_host() - ref).max() / np.abs(ref).max()
    assert err <= 1e-14, err
    rerr = np.abs(T.rhs - g["raw_rhs"]).max() / np.abs(g["raw_rhs"]).max()
    assert rerr <= 1e-14, rerr


@pytest.mark.parametrize("name", CASES)
def test_hierarchy_levels(name):
    c, z, mesh, cm, groups, basis, T = host_setup(name)
    N = basis.size
    pidx = PieceIndex.build(cm.species_volume)
    lb = LevelBuilder(cm, basis)
    lvl = aggregation_level_data(lb, groups[0])
    R0 = initial_restriction(lvl, {(int(j), int(s)): b for b, (j, s) in enumerate(pidx.pieces)}, N)
    M = host_galerkin(T.row_ptr, T.col, T.evaluate_host(), R0)
    b = restrict_rhs(R0, T.rhs, lvl.num_blocks, N)
    fine = lvl
    for lam in range(1, c.num_levels + 1):
        p = f"L{lam}_"
        assert np.array_equal(M[0], z[p + "row_ptr"]) and np.array_equal(M[1], z[p + "col"])
        ref = fixture_array(z, p + "val")
        err = np.abs(M[2] - ref).max() / np.abs(ref).max()
        assert err <= TOL[name], (lam, err)
        assert np.abs(b - z[p + "rhs"]).max() <= 1e-13 * np.abs(z[p + "rhs"]).max()
        gph = aggregate_graph(fine, mesh)
        adj = np.array([v for a in gph.adjacency for v in a], np.int64)
        assert np.array_equal(adj, z[p + "adj"])
        if lam < c.num_levels:
            R, coarse = build_restriction(lb, fine, groups[lam])
            assert np.array_equal(R[1], z[p + "R_col"])
            assert np.abs(R[2] - fixture_array(z, p + "R_val")).max() <= 1e-12
            M = host_galerkin(*M, R)
            b = restrict_rhs(R, b, coarse.num_blocks, N)
            fine = coarse
