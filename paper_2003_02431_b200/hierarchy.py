"""Hierarchy containers the solvers read (duck-types of cutdg
`HierarchyLevel` / `MultigridHierarchy`, transfer.py:408-453, and
`MeshGraph`, mesh.py:97-116) plus a loader for serialized hierarchies.

The setup that *builds* a hierarchy (cut-cell geometry, SIP assembly,
aggregation bases, Galerkin products) is out of this round's scope
(SURVEY.md 8(f) rows 1-3); solvers accept either the reference's own
hierarchy objects (cutdg.bench.assemble_case(...).hierarchy) or one loaded
from an .npz written by tests/golden/make_golden.py (same arrays: BSR of
every level matrix and restriction, right-hand sides, aggregate graphs).
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .blockmatrix import BlockSparseMatrix, uniform_layout
from .errors import DimensionMismatchError


@dataclass(frozen=True)
class MeshGraph:
    num_cells: int
    edges: tuple
    adjacency: tuple
    # (ptr int64[n+1], col int64[nnz]): the adjacency with every row sorted,
    # when the builder has it as arrays (schwarz_partition reads it instead
    # of flattening `adjacency`); None for graphs built elsewhere
    csr: object = field(default=None, compare=False, repr=False)


def graph_csr(rows: np.ndarray, cols: np.ndarray, n: int):
    """(ptr, col) of the directed pairs (rows, cols), rows sorted, each row's
    columns sorted (duplicates kept, like sorted(adjacency[i]))."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    o = np.lexsort((cols, rows))
    ptr = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=ptr[1:])
    return ptr, np.ascontiguousarray(cols[o])


@dataclass(frozen=True)
class _Basis:
    degree: int
    dim: int

    @property
    def size(self) -> int:
        from math import comb

        return comb(self.degree + self.dim, self.dim)


@dataclass(frozen=True)
class LevelInfo:
    """What the solvers read of cutdg LevelData (transfer.py:57-94)."""

    basis: _Basis
    num_blocks: int

    @property
    def block_size(self) -> int:
        return self.basis.size

    @property
    def num_dofs(self) -> int:
        return self.num_blocks * self.block_size

    @property
    def aggregates(self):  # duck-type marker used by schwarz._Nodes
        return range(self.num_blocks)


@dataclass
class HierarchyLevel:
    data: LevelInfo
    matrix: BlockSparseMatrix
    rhs: Optional[np.ndarray]
    restriction: Optional[BlockSparseMatrix]
    graph: MeshGraph

    @property
    def num_dofs(self) -> int:
        return self.data.num_dofs


@dataclass
class MultigridHierarchy:
    levels: list
    meta: dict
    to_level1: object = None  # R0: raw (cell, species) blocks -> level-1 aggregates

    @property
    def num_levels(self) -> int:
        return len(self.levels)

    def level(self, lam: int) -> HierarchyLevel:
        if not 1 <= lam <= len(self.levels):
            raise DimensionMismatchError(f"no level {lam}")
        return self.levels[lam - 1]


def _graph(ptr: np.ndarray, adj: np.ndarray) -> MeshGraph:
    n = len(ptr) - 1
    adjacency = tuple(tuple(int(v) for v in adj[ptr[i]:ptr[i + 1]]) for i in range(n))
    edges = tuple(sorted((a, b) for a in range(n) for b in adjacency[a] if a < b))
    ptr = np.asarray(ptr, np.int64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ptr))
    return MeshGraph(num_cells=n, edges=edges, adjacency=adjacency,
                     csr=graph_csr(rows, np.asarray(adj, np.int64)[ptr[0]:ptr[-1]], n))


def fixture_array(z, key: str) -> np.ndarray:
    """z[key], reassembling block arrays stored deduplicated
    (key__uniq[key__idx], tests/golden/dedup_fixture.py)."""
    if key in z.files:
        return z[key]
    return z[key + "__uniq"][z[key + "__idx"]]


def fixture_has(z, key: str) -> bool:
    return key in z.files or (key + "__uniq") in z.files


def load_hierarchy(path_or_npz, num_levels: Optional[int] = None) -> MultigridHierarchy:
    """Rebuild a hierarchy from a fixture written by make_golden.py."""
    z = np.load(path_or_npz) if isinstance(path_or_npz, str) else path_or_npz
    meta = json.loads(bytes(z["meta"]).decode())
    dim = int(meta["dim"])
    L = int(meta["num_levels"]) if num_levels is None else num_levels
    levels = []
    for lam in range(1, L + 1):
        p = f"L{lam}_"
        N = int(z[p + "N"])
        rp, col, val = z[p + "row_ptr"], z[p + "col"], fixture_array(z, p + "val")
        nb = len(rp) - 1
        lay = uniform_layout(nb, N)
        M = BlockSparseMatrix.from_bsr(rp, col, val, lay, lay)
        R = None
        if lam < L and (p + "R_row_ptr") in z.files:
            nc = int(z[p + "R_ncols"])
            R = BlockSparseMatrix.from_bsr(z[p + "R_row_ptr"], z[p + "R_col"],
                                           fixture_array(z, p + "R_val"), lay,
                                           uniform_layout(nc, N))
        info = LevelInfo(basis=_Basis(int(z[p + "degree"]), dim), num_blocks=nb)
        levels.append(HierarchyLevel(data=info, matrix=M, rhs=np.array(z[p + "rhs"]),
                                     restriction=R,
                                     graph=_graph(z[p + "adj_ptr"], z[p + "adj"])))
    return MultigridHierarchy(levels=levels, meta=meta)
