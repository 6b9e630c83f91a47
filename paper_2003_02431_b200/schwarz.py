"""Overlapping Schwarz partition (host setup) -- drop-in for cutdg
`SchwarzPartition` / `schwarz_partition` (solvers.py:312-457).

The partition must be reproduced exactly for parity: greedy
breadth-first cores seeded at the lowest unassigned node, neighbours queued
in ascending order, a core closes once it holds >= target DOFs, then every
core grows by one neighbour layer; damping[dof] counts the extended blocks
containing the DOF.  The device side (pmg.PmgPlan over all extended blocks)
is built lazily from `block_rows` and cached in `cache`.
"""
from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field

import numpy as np

from .errors import DimensionMismatchError, InvalidConfigError


@dataclass
class SchwarzPartition:
    """Disjoint cores, their one-layer extensions (`blocks`), the matrix
    block rows of every extension, and the per-DOF overlap damping."""

    cores: tuple
    blocks: tuple
    block_rows: tuple
    damping: np.ndarray
    dim: int
    cache: dict = field(default_factory=dict)

    @property
    def num_blocks(self) -> int:
        return len(self.blocks)


class _Nodes:
    """Uniform view of the two index structures the reference accepts
    (solvers.py:330-381): a raw species index map (nodes = background cells,
    each owning one or two species blocks) or an aggregation level (nodes =
    aggregates, one block each)."""

    def __init__(self, indexmap):
        self.uniform_level = False
        if hasattr(indexmap, "block_of"):  # raw XdgIndexMap
            imap = indexmap
            self.num_nodes = imap.cutmesh.mesh.num_cells
            self.dim = imap.cutmesh.mesh.dim
            per = [[] for _ in range(self.num_nodes)]
            for b, (cell, _s) in enumerate(imap.blocks):
                per[cell].append(b)
            self._blocks = [tuple(p) for p in per]
            self._slices = [imap.block_slice(b) for b in range(len(imap.blocks))]
            self.total = imap.L
        elif hasattr(indexmap, "aggregates") or hasattr(indexmap, "num_blocks"):
            lvl = indexmap
            self.num_nodes = lvl.num_blocks
            size = lvl.block_size
            self.dim = lvl.basis.dim
            self._blocks = self._slices = None  # node g = block g (no lists)
            self.total = lvl.num_dofs
            self.block_size = size
            self.uniform_level = True
        else:
            raise InvalidConfigError(
                "index structure must be a species index map or a level")

    def blocks_of(self, j):
        if self.uniform_level:
            return (j,)
        return self._blocks[j]

    def dofs_of(self, j):
        if self.uniform_level:
            return self.block_size
        return sum(self._slices[b].stop - self._slices[b].start
                   for b in self._blocks[j])

    def dof_slices(self, j):
        if self.uniform_level:
            return [slice(j * self.block_size, (j + 1) * self.block_size)]
        return [self._slices[b] for b in self._blocks[j]]


def schwarz_partition(mesh_graph, indexmap, target_dofs: int) -> SchwarzPartition:
    nodes = _Nodes(indexmap)
    n = nodes.num_nodes
    if mesh_graph.num_cells != n:
        raise DimensionMismatchError(
            "graph and index structure disagree on the cell count")
    if nodes.uniform_level:
        dofs = np.full(n, nodes.block_size, np.int64)
    else:
        dofs = np.array([nodes.dofs_of(j) for j in range(n)], np.int64)
    largest = int(dofs.max()) if n else 0
    if target_dofs < largest:
        raise InvalidConfigError(
            f"target {target_dofs} below the largest cell ({largest} DOFs)")
    if nodes.uniform_level:
        return _schwarz_partition_native(mesh_graph, nodes, dofs, int(target_dofs))
    nbrs = [sorted(a) for a in mesh_graph.adjacency]

    taken = np.zeros(n, bool)
    cores = []
    next_free = 0
    while True:
        while next_free < n and taken[next_free]:
            next_free += 1
        if next_free == n:
            break
        core, acc = [], 0
        frontier = deque([next_free])
        seen = {next_free}
        while frontier and acc < target_dofs:
            c = frontier.popleft()
            if taken[c]:
                continue
            taken[c] = True
            core.append(c)
            acc += int(dofs[c])
            for nb in nbrs[c]:
                if not taken[nb] and nb not in seen:
                    seen.add(nb)
                    frontier.append(nb)
        cores.append(tuple(sorted(core)))

    extended = []
    for core in cores:
        grown = set(core)
        for c in core:
            grown.update(nbrs[c])
        extended.append(tuple(sorted(grown)))

    damping = np.zeros(nodes.total)
    for ext in extended:
        for c in ext:
            for sl in nodes.dof_slices(c):
                damping[sl] += 1.0
    if np.any(damping < 1.0):
        raise InvalidConfigError("partition left degrees of freedom uncovered")

    block_rows = tuple(tuple(sorted(b for c in ext for b in nodes.blocks_of(c)))
                       for ext in extended)
    return SchwarzPartition(cores=tuple(cores), blocks=tuple(extended),
                            block_rows=block_rows, damping=damping,
                            dim=nodes.dim)


def _pieces(flat: np.ndarray, ptr: np.ndarray) -> list:
    """[flat[ptr[q]:ptr[q+1]] as a list of Python ints for each q]."""
    vals = flat[:int(ptr[-1])].tolist()
    p = ptr.tolist()
    return [vals[p[q]:p[q + 1]] for q in range(len(p) - 1)]


def _schwarz_partition_native(mesh_graph, nodes, dofs, target: int) -> SchwarzPartition:
    """schwarz_partition on an aggregation level (node g = block g of
    block_size DOFs) through the native xdg_schwarz_partition: the same
    greedy BFS cores and one-layer extension, then damping and block rows
    vectorised."""
    from . import _native as nat

    n = nodes.num_nodes
    csr = getattr(mesh_graph, "csr", None)
    if csr is not None and (len(csr[0]) != n + 1 or int(csr[0][-1]) != sum(
            len(a) for a in mesh_graph.adjacency)):
        csr = None  # stale copy (graph rebuilt with another adjacency): flatten
    if csr is not None:  # sorted rows built from the builder's arrays
        ptr, flat = csr
        ptr = np.ascontiguousarray(ptr, np.int64)
        flat = np.ascontiguousarray(flat, np.int64)
    else:
        adj = [sorted(a) for a in mesh_graph.adjacency]
        ptr = np.zeros(n + 1, np.int64)
        np.cumsum([len(a) for a in adj], out=ptr[1:])
        flat = np.ascontiguousarray(np.fromiter((v for a in adj for v in a), np.int64,
                                                count=int(ptr[-1])))
    dofs = np.ascontiguousarray(dofs, np.int64)
    lib = nat.load()
    ncore = int(lib.xdg_schwarz_partition(n, ptr.ctypes.data, flat.ctypes.data,
                                          dofs.ctypes.data, target))
    sz = np.zeros(2, np.int64)
    lib.xdg_schwarz_sizes(sz.ctypes.data)
    cptr, cnodes = np.zeros(ncore + 1, np.int64), np.zeros(max(int(sz[0]), 1), np.int64)
    eptr, enodes = np.zeros(ncore + 1, np.int64), np.zeros(max(int(sz[1]), 1), np.int64)
    lib.xdg_schwarz_copy(cptr.ctypes.data, cnodes.ctypes.data, eptr.ctypes.data,
                         enodes.ctypes.data)
    cores = tuple(map(tuple, _pieces(cnodes, cptr)))
    extended = tuple(map(tuple, _pieces(enodes, eptr)))
    N = nodes.block_size
    cover = np.bincount(enodes[:int(eptr[-1])], minlength=n).astype(float)
    damping = np.repeat(cover, N)
    if np.any(damping < 1.0):
        raise InvalidConfigError("partition left degrees of freedom uncovered")
    return SchwarzPartition(cores=cores, blocks=extended, block_rows=extended,
                            damping=damping, dim=nodes.dim)
