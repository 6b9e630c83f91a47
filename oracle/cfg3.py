"""Exact numpy recipe of the BASELINE config-3 synthetic block-MSR operator
(SURVEY.md 8(d) "Exact recipes") -- TEST INFRASTRUCTURE.

rng = default_rng(seed); cut = rng.choice(J, round(0.05 J), replace=False);
pattern in (row, col) order; values: A = rng.standard_normal((nbr, N, N)),
diagonal blocks A^T A + 10 I in block-row order, then off-diagonal blocks
0.1 * rng.standard_normal((n_off, N, N)) in sorted order;
x = default_rng(1).standard_normal(L).  At 10^3 the resulting CSR equals the
reference's BlockSparseMatrix.tocsr() bit for bit (survey-verified; re-pinned
by tests/test_oracle.py against the reference-built fixture).
"""
from __future__ import annotations

import numpy as np


def build(n: int, seed: int = 0, N: int = 10, frac: float = 0.05):
    """Returns (row_ptr, col, val[nnzb, N, N] row-major, x)."""
    J = n ** 3
    rng = np.random.default_rng(seed)
    cut = np.zeros(J, bool)
    cut[rng.choice(J, size=int(round(frac * J)), replace=False)] = True
    first = np.concatenate([[0], np.cumsum(1 + cut.astype(np.int64))])
    j = np.arange(J, dtype=np.int64)
    rows = [first[:-1], first[:-1][cut] + 1, first[:-1][cut], first[:-1][cut] + 1]
    cols = [first[:-1], first[:-1][cut] + 1, first[:-1][cut] + 1, first[:-1][cut]]
    coords = (j % n, (j // n) % n, j // (n * n))
    for c, stride in zip(coords, (1, n, n * n)):
        for sgn in (-1, 1):
            ok = (c + sgn >= 0) & (c + sgn < n)
            a = j[ok]
            b = a + sgn * stride
            rows.append(first[a])
            cols.append(first[b])
            both = cut[a] & cut[b]
            rows.append(first[a[both]] + 1)
            cols.append(first[b[both]] + 1)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    order = np.lexsort((cols, rows))
    rows, cols = rows[order], cols[order]
    nbr = int(first[-1])
    is_diag = rows == cols
    A = rng.standard_normal((nbr, N, N))
    val = np.empty((len(rows), N, N))
    val[is_diag] = np.einsum("kji,kjl->kil", A, A) + 10.0 * np.eye(N)
    val[~is_diag] = 0.1 * rng.standard_normal((int((~is_diag).sum()), N, N))
    row_ptr = np.zeros(nbr + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=nbr), out=row_ptr[1:])
    x = np.random.default_rng(1).standard_normal(nbr * N)
    return row_ptr, cols, val, x
