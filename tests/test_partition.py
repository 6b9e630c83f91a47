"""Host-side Schwarz partition (solvers.py:384-457 restated in
paper_2003_02431_b200/schwarz.py) reproduces the reference's partitions
exactly on every golden hierarchy level."""
import numpy as np
import pytest

from conftest import golden_path
from paper_2003_02431_b200.errors import InvalidConfigError
from paper_2003_02431_b200.hierarchy import load_hierarchy
from paper_2003_02431_b200.schwarz import schwarz_partition


def ragged(ptr, flat):
    return [tuple(int(v) for v in flat[ptr[i]:ptr[i + 1]]) for i in range(len(ptr) - 1)]


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3"])
def test_partition_matches_reference(case):
    z = np.load(golden_path(case))
    hier = load_hierarchy(z)
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        for key in z.files:
            if key.startswith(f"L{lam}_T") and key.endswith("_damping"):
                tgt = int(key[len(f"L{lam}_T"):].split("_")[0])
                q = f"L{lam}_T{tgt}_"
                part = schwarz_partition(lv.graph, lv.data, max(tgt, lv.data.block_size))
                assert list(part.cores) == ragged(z[q + "cores_ptr"], z[q + "cores"])
                assert list(part.block_rows) == ragged(z[q + "rows_ptr"], z[q + "rows"])
                assert np.array_equal(part.damping, z[q + "damping"])


def test_partition_rejects_target_below_cell():
    hier = load_hierarchy(np.load(golden_path("bench4")))
    lv = hier.level(1)
    with pytest.raises(InvalidConfigError):
        schwarz_partition(lv.graph, lv.data, lv.data.block_size - 1)


@pytest.mark.parametrize("case", ["bench4", "cfg1", "sphere8p3"])
def test_partition_graph_csr_same_as_adjacency(case):
    """The graph's array copy (MeshGraph.csr) is the sorted adjacency, and
    the partition read through it equals the one read from the tuples."""
    from dataclasses import replace

    hier = load_hierarchy(np.load(golden_path(case)))
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        ptr, flat = lv.graph.csr
        srt = [v for a in lv.graph.adjacency for v in sorted(a)]
        assert flat.tolist() == srt
        assert np.diff(ptr).tolist() == [len(a) for a in lv.graph.adjacency]
        tgt = max(2000, lv.data.block_size)
        a = schwarz_partition(lv.graph, lv.data, tgt)
        b = schwarz_partition(replace(lv.graph, csr=None), lv.data, tgt)
        assert a.cores == b.cores and a.block_rows == b.block_rows
        assert np.array_equal(a.damping, b.damping)


@pytest.mark.parametrize("case", ["cfg1", "sphere8p3"])
def test_array_form_transpose_matches_dict_transpose(case):
    """BlockSparseMatrix.transpose on array-form operators (one stable sort)
    gives the same blocks as the reference's dict loop (blockmatrix.py:
    127-131) -- the restrictions R of every level and the level matrices."""
    from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix

    hier = load_hierarchy(np.load(golden_path(case)))
    for lam in range(1, hier.num_levels + 1):
        lv = hier.level(lam)
        for M in (lv.matrix, lv.restriction):
            if M is None:
                continue
            rp, col, val = M.bsr_arrays()
            A = BlockSparseMatrix.from_bsr(rp, col, val, M.row_layout, M.col_layout)
            T = A.transpose()
            assert T._blocks is None  # array form kept
            Bd = BlockSparseMatrix(M.row_layout, M.col_layout)
            for k in range(len(rp) - 1):
                for j in range(rp[k], rp[k + 1]):
                    Bd.add_block(k, int(col[j]), val[j])
            ref = Bd.transpose()
            t_rp, t_col, t_val = T.bsr_arrays()
            r_rp, r_col, r_val = ref.bsr_arrays()
            assert np.array_equal(t_rp, r_rp) and np.array_equal(t_col, r_col)
            assert np.array_equal(t_val, r_val)
