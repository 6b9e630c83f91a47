"""Drop-in for the transfer operations of the solver path
(cutdg transfer.py:344-351 galerkin_restrict, 408-453 containers).

`galerkin_restrict(M, b, R)` = (R^T M R, R^T b): the Galerkin coarse operator
(the paper's Table-2 "matrix-matrix" product).  The
symbolic phase (output pattern, per-output term lists) is vectorised on the
host; the numeric phase is the xdg_galerkin kernel (one CTA per coarse
block, terms R_i^T M_ik R_k accumulated in a fixed order).  R x_c and R^T r
of the solvers (solvers.py:730,734) are device BSR SpMVs.
"""
from __future__ import annotations

import numpy as np
import scipy.linalg  # noqa: F401  (imported before worker processes fork)
import torch

from . import _native as nat
from .blockmatrix import BlockSparseMatrix, as_block_sparse
from .errors import LayoutMismatchError
from .hierarchy import HierarchyLevel, LevelInfo, MeshGraph, MultigridHierarchy  # noqa: F401
from .hierarchy import graph_csr

I32 = torch.int32


def galerkin_symbolic(rp, col, R_rp, R_col, n_coarse):
    """Pattern of R^T M R and its term lists.  Requires one R block per fine
    row.  Returns (Mc_row_ptr, Mc_col, tptr, t_e, t_ri, t_rk)."""
    rp, col = np.asarray(rp, np.int64), np.asarray(col, np.int64)
    R_rp, R_col = np.asarray(R_rp, np.int64), np.asarray(R_col, np.int64)
    if not np.all(np.diff(R_rp) == 1):
        raise LayoutMismatchError("Galerkin product expects one R block per fine row")
    parent = R_col
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    G, H = parent[rows], parent[col]
    order = np.lexsort((col, rows, H, G))          # (G, H, i, k)
    key = G[order] * n_coarse + H[order]
    first = np.flatnonzero(np.r_[True, key[1:] != key[:-1]]) if len(key) else np.zeros(0, np.int64)
    tptr = np.r_[first, len(key)]
    uk = key[first]
    c_rows, c_cols = uk // n_coarse, uk % n_coarse
    c_rp = np.zeros(n_coarse + 1, np.int64)
    np.cumsum(np.bincount(c_rows, minlength=n_coarse), out=c_rp[1:])
    return c_rp, c_cols, tptr, order, rows[order], col[order]


def galerkin_device(M, R):
    """Mc = R^T M R on the device.  M, R: BlockSparseMatrix (ours or the
    reference's); returns (DeviceBSR of Mc, host (row_ptr, col))."""
    from .device import Context, DeviceBSR

    M, R = as_block_sparse(M), as_block_sparse(R)
    ctx = Context.get()
    Md, Rd = M.device(ctx), R.device(ctx)
    return galerkin_dev(Md, Rd, R.col_layout.num_blocks, ctx)


def galerkin_dev(Md, Rd, nc, ctx, pattern=None, r_pattern=None):
    """R^T M R for device operands (DeviceBSR).  `pattern` / `r_pattern`:
    host copies of (row_ptr, col) when the caller has them."""
    from .device import DeviceBSR

    if Md.N != Rd.N:
        raise LayoutMismatchError("M and R block sizes differ")
    if pattern is None:
        pattern = (Md.row_ptr.cpu().numpy(), Md.col.cpu().numpy())
    if r_pattern is None:
        r_pattern = (Rd.row_ptr.cpu().numpy(), Rd.col.cpu().numpy())
    c_rp, c_col, tptr, te, tri, trk = galerkin_symbolic(
        pattern[0], pattern[1], r_pattern[0], r_pattern[1], nc)
    dev = ctx.device
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev, I32)  # noqa: E731
    N = Md.N
    out = torch.empty(len(c_col), N, N, dtype=torch.float64, device=dev)
    targs = [up(tptr), up(te), up(tri), up(trk)]
    nat.check(ctx.lib.xdg_galerkin(len(c_col), N, *[t.data_ptr() for t in targs],
                                   Md.val_t.data_ptr(), Rd.val_t.data_ptr(),
                                   out.data_ptr(), ctx.stream), "galerkin")
    C = DeviceBSR(nc, nc, N, up(c_rp), up(c_col), out, ctx)
    return C, (c_rp, c_col)


def galerkin_restrict(M, b, R) -> tuple:
    """Coarse system (R^T M R, R^T b) (transfer.py:344-351)."""
    R = getattr(R, "matrix", R)
    Rb = as_block_sparse(R)
    C, (c_rp, c_col) = galerkin_device(M, Rb)
    rp, col, val = C.to_host_rowmajor()
    Mc = BlockSparseMatrix.from_bsr(c_rp, c_col, val, Rb.col_layout, Rb.col_layout)
    Mc._dev, Mc._dev_pad = C, None
    bc = None
    if b is not None:
        Rt = Rb.transpose()
        bc = Rt.matvec(np.asarray(b, dtype=float))
    return Mc, bc


# ===========================================================================
# Level construction: aggregate carriers, restrictions and
# the Galerkin hierarchy of build_hierarchy (transfer.py:107-341, 456-522 of
# the reference).  Host work is per *cut* aggregate; aggregates made only of
# uncut pieces are translation invariant on the uniform mesh, so their
# carriers and restriction blocks are computed once per relative shape and
# reused (identical up to roundoff to the reference's per-aggregate
# computation).  The Galerkin products run on the device (xdg_galerkin) and
# the raw operator is formed on the device (xdg_assemble_blocks).

GRAM_PIVOT_RTOL = 1e-13


def _monomial_values(points, lo, hi, dim, degree):
    """transfer.py:114-130."""
    from .assembly import multi_indices

    center = 0.5 * (lo + hi)
    halfwidth = 0.5 * (hi - lo)
    t = (points - center) / halfwidth
    exps = multi_indices(degree, dim)
    pw = [[None] + [t[:, d] ** e for e in range(1, degree + 1)] for d in range(dim)]
    out = np.empty((len(points), len(exps)))
    for m, a in enumerate(exps):
        col = np.ones(len(points))
        for d, e in enumerate(a):
            if e:
                col *= pw[d][e]
        out[:, m] = col
    return out


def _chol_or_degenerate(G, context):
    """transfer.py:133-149."""
    from .errors import DegenerateAggregateError

    n = len(G)
    L = np.zeros_like(G)
    threshold = GRAM_PIVOT_RTOL * float(np.max(np.diag(G)))
    for i in range(n):
        s = G[i, i] - L[i, :i] @ L[i, :i]
        if not s > threshold:
            raise DegenerateAggregateError(
                f"aggregate Gram pivot {s:.3e} below threshold {threshold:.3e} ({context})")
        L[i, i] = np.sqrt(s)
        if i + 1 < n:
            L[i + 1:, i] = (G[i + 1:, i] - L[i + 1:, :i] @ L[i, :i]) / L[i, i]
    return L


class LevelBuilder:
    """Carriers and transfer blocks of one cut-cell mesh (transfer.py:152-341).
    Per-aggregate work runs in forked worker processes (_pool.fork_map); the
    mass matrices of cut pieces are computed once and shared by all levels."""

    def __init__(self, cm, basis, workers=None):
        self.cm, self.basis = cm, basis
        self.mesh = cm.mesh
        self.N = basis.size
        self.workers = workers
        self._carrier_cache: dict = {}
        self._block_cache: dict = {}
        self.mass: dict = {}
        self.cache_hits = 0

    def uncut(self, p) -> bool:
        return (int(p[0]), int(p[1])) not in self.cm.cut_volume_rules

    def _shape_key(self, pieces):
        m = self.mesh.multi(np.array([j for j, _ in pieces]))
        return tuple(map(tuple, (m - m.min(axis=0)).tolist()))

    def _bbox(self, pieces):
        lo, hi = self.mesh.bounds(np.array([j for j, _ in pieces]))
        return lo.min(axis=0), hi.max(axis=0)

    def _cell_monomial_coefficients(self, j, lo, hi):
        from .cutcells import tensor_rule

        clo, chi = self.mesh.bounds(j)
        rule = tensor_rule(clo, chi, self.basis.degree + 1)
        vals = self.basis.eval(clo, chi, rule.nodes)
        mono = _monomial_values(rule.nodes, lo, hi, self.mesh.dim, self.basis.degree)
        return vals.T @ (mono * rule.weights[:, None])

    def _carrier_exact(self, pieces):
        """build_carrier (transfer.py:170-205)."""
        from scipy.linalg import solve_triangular

        from .cutcells import quad_volume

        dim, deg, n = self.mesh.dim, self.basis.degree, self.N
        lo, hi = self._bbox(pieces)
        G = np.zeros((n, n))
        for j, s in pieces:
            rule = quad_volume(self.cm, j, s)
            mono = _monomial_values(rule.nodes, lo, hi, dim, deg)
            G += mono.T @ (mono * rule.weights[:, None])
        ctx = f"pieces {tuple(pieces)}"
        L1 = _chol_or_degenerate(0.5 * (G + G.T), ctx)
        T = solve_triangular(L1, np.eye(n), lower=True).T
        G2 = T.T @ G @ T
        L2 = _chol_or_degenerate(0.5 * (G2 + G2.T), ctx)
        T = T @ solve_triangular(L2, np.eye(n), lower=True).T
        out = np.empty((len(pieces) * n, n))
        for i, (j, _s) in enumerate(pieces):
            out[i * n:(i + 1) * n] = self._cell_monomial_coefficients(j, lo, hi) @ T
        return out

    def _mass_exact(self, p):
        """_piece_plain_mass (transfer.py:267-278) of a cut piece."""
        j, s = p
        rule = self.cm.cut_volume_rules[(j, s)]
        lo, hi = self.mesh.bounds(j)
        vals = self.basis.eval(lo, hi, rule.nodes)
        return vals.T @ (vals * rule.weights[:, None])

    def piece_mass(self, p):
        """None = identity (uncut piece)."""
        if self.uncut(p):
            return None
        m = self.mass.get(p)
        if m is None:
            m = self.mass[p] = self._mass_exact(p)
        return m

    def precompute_masses(self):
        from ._pool import fork_map

        todo = sorted(k for k in self.cm.cut_volume_rules if k not in self.mass)
        for p, m in zip(todo, fork_map(_mass_job, todo, {"lb": self}, self.workers)):
            self.mass[p] = m


def _mass_job(p):
    from ._pool import STATE

    return STATE["lb"]._mass_exact(p)


def _carrier_job(pieces):
    from ._pool import STATE

    return STATE["lb"]._carrier_exact(pieces)


def _restriction_job(job):
    """Carrier of one coarse aggregate and its blocks against every fine
    member (transfer.py:318-334)."""
    from ._pool import STATE

    lb, fine = STATE["lb"], STATE["fine"]
    pieces, members = job
    n = lb.N
    carrier = lb._carrier_exact(pieces)
    pos = {p: i for i, p in enumerate(pieces)}
    blocks = []
    for g in members:
        block = np.zeros((n, n))
        fc = fine.carriers[g]
        for i, p in enumerate(fine.aggregates[g]):
            left = _rows(fc, i, n)
            right = carrier[pos[p] * n:(pos[p] + 1) * n]
            mass = lb.piece_mass(p)
            block += left.T @ right if mass is None else left.T @ mass @ right
        blocks.append(block)
    return carrier, blocks


class LevelData:
    """Aggregates (tuples of pieces) and carriers (None = identity) of one
    level (transfer.py:57-94)."""

    def __init__(self, aggregates, carriers):
        self.aggregates = aggregates
        self.carriers = carriers

    @property
    def num_blocks(self):
        return len(self.aggregates)


def aggregation_level_data(lb: LevelBuilder, groups) -> LevelData:
    """transfer.py:208-236: uncut singletons keep the background basis."""
    from ._pool import fork_map

    aggs, carriers, todo, where = [], [], [], {}
    for g in groups:
        pieces = tuple((int(j), int(s)) for j, s in sorted(g))
        aggs.append(pieces)
        if len(pieces) == 1 and lb.uncut(pieces[0]):
            carriers.append(None)
            continue
        key = lb._shape_key(pieces) if all(lb.uncut(p) for p in pieces) else None
        if key is not None and (key in lb._carrier_cache or key in where):
            lb.cache_hits += 1
            carriers.append(("key", key))
            continue
        if key is not None:
            where[key] = len(todo)
        carriers.append(("job", len(todo)))
        todo.append(pieces)
    res = fork_map(_carrier_job, todo, {"lb": lb}, lb.workers)
    for key, i in where.items():
        lb._carrier_cache[key] = res[i]
    out = []
    for c in carriers:
        if c is None:
            out.append(None)
        elif c[0] == "job":
            out.append(res[c[1]])
        else:
            out.append(lb._carrier_cache[c[1]])
    return LevelData(aggs, out)


def _rows(carrier, i, n):
    return np.eye(n) if carrier is None else carrier[i * n:(i + 1) * n]


def initial_restriction(level: LevelData, block_of, n):
    """transfer.py:239-264 as BSR arrays (one block per raw row).
    block_of[(j, s)] -> raw block index."""
    nb = sum(len(a) for a in level.aggregates)
    col = np.empty(nb, np.int64)
    val = np.empty((nb, n, n))
    for G, pieces in enumerate(level.aggregates):
        c = level.carriers[G]
        for i, p in enumerate(pieces):
            b = block_of[p]
            col[b] = G
            val[b] = _rows(c, i, n)
    return np.arange(nb + 1, dtype=np.int64), col, val


def build_restriction(lb: LevelBuilder, fine: LevelData, coarse_groups):
    """transfer.py:281-341: returns ((row_ptr, col, val) over fine
    aggregates, coarse LevelData).  Coarse aggregates made of uncut pieces
    are computed once per (shape, member partition) class."""
    from ._pool import fork_map

    from .errors import InvalidMapError

    n = lb.N
    p2f = {}
    for g, pieces in enumerate(fine.aggregates):
        for p in pieces:
            p2f[p] = g
    nf = fine.num_blocks
    plan, todo, pending = [], [], {}
    lb.precompute_masses()
    for G, group in enumerate(coarse_groups):
        pieces = tuple((int(j), int(s)) for j, s in sorted(group))
        members = sorted({p2f[p] for p in pieces})
        if sum(len(fine.aggregates[g]) for g in members) != len(pieces):
            raise InvalidMapError(
                f"coarse aggregation map splits a fine aggregate (coarse group {pieces})")
        if len(members) == 1:
            plan.append((pieces, members, "inherit", None))
            continue
        key = None
        if all(lb.uncut(p) for p in pieces):
            pos = {p: i for i, p in enumerate(pieces)}
            key = (lb._shape_key(pieces),
                   tuple(tuple(pos[p] for p in fine.aggregates[g]) for g in members))
            if key in lb._block_cache or key in pending:
                lb.cache_hits += 1
                plan.append((pieces, members, "cache", key))
                continue
            pending[key] = len(todo)
        plan.append((pieces, members, "job", len(todo)))
        todo.append((pieces, members))
    res = fork_map(_restriction_job, todo, {"lb": lb, "fine": fine}, lb.workers)
    for key, i in pending.items():
        lb._block_cache[key] = res[i]
        lb._carrier_cache.setdefault(key[0], res[i][0])
    col = np.empty(nf, np.int64)
    val = np.empty((nf, n, n))
    aggs, carriers = [], []
    for G, (pieces, members, how, ref) in enumerate(plan):
        aggs.append(pieces)
        if how == "inherit":
            carriers.append(fine.carriers[members[0]])
            col[members[0]] = G
            val[members[0]] = np.eye(n)
            continue
        carrier, blocks = res[ref] if how == "job" else lb._block_cache[ref]
        carriers.append(carrier)
        for g, blk in zip(members, blocks):
            col[g] = G
            val[g] = blk
    return (np.arange(nf + 1, dtype=np.int64), col, val), LevelData(aggs, carriers)


def aggregate_graph(level: LevelData, mesh) -> MeshGraph:
    """aggregate_block_graph (transfer.py:377-406): aggregates sharing a
    cell, or owning face-neighbour cells, are adjacent."""
    J = mesh.num_cells
    own = np.full((J, 2), -1, np.int64)
    for g, pieces in enumerate(level.aggregates):
        for j, s in pieces:
            own[j, s] = g
    pairs = []
    both = (own[:, 0] >= 0) & (own[:, 1] >= 0) & (own[:, 0] != own[:, 1])
    pairs.append(np.sort(own[both], axis=1))
    adj = mesh.adjacency()
    ea = np.repeat(np.arange(J), [len(a) for a in adj])
    eb = np.array([b for a in adj for b in a], np.int64)
    keep = ea < eb
    ea, eb = ea[keep], eb[keep]
    for x in (0, 1):
        for y in (0, 1):
            A, Bq = own[ea, x], own[eb, y]
            ok = (A >= 0) & (Bq >= 0) & (A != Bq)
            pairs.append(np.sort(np.stack([A[ok], Bq[ok]], axis=1), axis=1))
    P = np.unique(np.concatenate(pairs), axis=0) if pairs else np.zeros((0, 2), np.int64)
    n = level.num_blocks
    nbrs = [[] for _ in range(n)]
    for a, b in P.tolist():
        nbrs[a].append(b)
        nbrs[b].append(a)
    return MeshGraph(num_cells=n, edges=tuple(map(tuple, P.tolist())),
                     adjacency=tuple(tuple(sorted(x)) for x in nbrs),
                     csr=graph_csr(np.concatenate([P[:, 0], P[:, 1]]),
                                   np.concatenate([P[:, 1], P[:, 0]]), n))


def assemble_device(terms, ctx=None):
    """Raw operator of SipTerms formed in HBM by xdg_assemble_blocks."""
    from .device import Context, DeviceBSR

    ctx = ctx or Context.get()
    dev = ctx.device
    up32 = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)  # noqa: E731
    upf = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dev)  # noqa: E731
    N = terms.N
    nout = len(terms.col)
    tabs = upf(terms.tables.transpose(0, 2, 1)) if len(terms.tables) else upf(np.zeros((1, N, N)))
    dense = upf(terms.dense.transpose(0, 2, 1)) if len(terms.dense) else upf(np.zeros((1, N, N)))
    out = torch.empty(nout, N, N, dtype=torch.float64, device=dev)
    args = [up32(terms.tptr), up32(terms.tid), upf(terms.coef), tabs, up32(terms.dptr),
            up32(terms.didx), dense]
    nat.check(ctx.lib.xdg_assemble_blocks(nout, N, *[a.data_ptr() for a in args],
                                          out.data_ptr(), ctx.stream), "assemble_blocks")
    return DeviceBSR(terms.nblocks, terms.nblocks, N, up32(terms.row_ptr), up32(terms.col),
                     out, ctx)


def restrict_rhs(R_bsr, b, n_coarse, N):
    """R^T b for a one-block-per-row R (row-major blocks)."""
    _, col, val = R_bsr
    out = np.zeros((n_coarse, N))
    np.add.at(out, col, np.einsum("bij,bi->bj", val, np.asarray(b).reshape(-1, N)))
    return out.reshape(-1)
