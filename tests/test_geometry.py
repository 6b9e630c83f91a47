"""Setup row SURVEY 8(f)#1: cut-cell classification and small-cell
agglomeration (paper_2003_02431_b200/geometry.py) against the reference's own
outputs (tests/golden/geo_*.npz, written by make_geometry_golden.py running
cutdg.cutcells.classify_and_build + agglomeration): species volumes equal to
the last bit, identical present-species sets, small-cell edges and level-1
aggregates (north_star: "must match the reference bit-exactly")."""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN
from paper_2003_02431_b200 import geometry as G

CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "geo_*.npz")))


def _build(z):
    dim, cells = int(z["dim"]), int(z["cells"])
    name = str(z["levelset"])
    params = {"center": tuple(z["center"]), "radius": float(z["radius"])} \
        if name == "sphere" else {}
    mesh = G.CartesianMesh([(-1.0, 1.0)] * dim, [cells] * dim)
    return mesh, G.level_set(name, params)


@pytest.mark.parametrize("case", CASES)
def test_classification_and_aggregates_match_reference(case):
    z = np.load(os.path.join(GOLDEN, f"{case}.npz"))
    mesh, phi = _build(z)
    vol = G.species_volumes(mesh, phi, int(z["quad_depth"]), int(z["gauss_order"]))
    ref = z["species_volume"]
    assert np.array_equal(vol > 0, ref > 0)            # present species per cell
    assert np.array_equal(vol, ref)                    # volumes, bit for bit
    edges = G.small_cell_pairs(vol, mesh.cell_volume, mesh.adjacency(), float(z["alpha"]))
    got = np.array(sorted((a[0], a[1], b[0], b[1]) for a, b in edges), np.int64).reshape(-1, 4)
    assert np.array_equal(got, z["small_edges"])
    def unpack(ptr, flat):
        return [[(int(p) // 2, int(p) % 2) for p in flat[ptr[i]:ptr[i + 1]]]
                for i in range(len(ptr) - 1)]

    aggs = G.aggregates(vol, edges)
    assert aggs == unpack(z["agg_ptr"], z["agg_pieces"])
    if "L2_agg_ptr" in z.files:       # multigrid levels 2..4
        levels = G.level_aggregates(mesh, vol, edges, 4)
        for lam in (2, 3, 4):
            assert levels[lam - 1] == unpack(z[f"L{lam}_agg_ptr"], z[f"L{lam}_agg_pieces"]), lam


def test_degenerate_level_set_raises():
    mesh = G.CartesianMesh([(-1.0, 1.0)] * 2, [2, 2])
    with pytest.raises(G.DegenerateLevelSetError):
        G.species_volumes(mesh, lambda x: np.zeros(len(x)), 3, 4)
