"""Fork-based process pool for the host side of setup: workers inherit the
large read-only state (cut-cell rules) instead of receiving it pickled; only
item descriptors and small result blocks cross process boundaries.  Results
come back in item order, independent of the split."""
from __future__ import annotations

import multiprocessing as mp
import os

import numpy as np

STATE: dict = {}
_FN = None


_LIMIT = None


def _init_worker():
    """One BLAS thread per worker: the workers already cover the cores."""
    global _LIMIT
    try:
        from threadpoolctl import threadpool_limits

        _LIMIT = threadpool_limits(1)
    except ImportError:  # pragma: no cover
        pass


def _chunk(chunk):
    return [_FN(it) for it in chunk]


def default_workers() -> int:
    return min(os.cpu_count() or 1, 32)


def fork_map(fn, items, state: dict, workers: int | None = None, min_items: int = 64):
    global _FN
    STATE.update(state)
    _FN = fn
    try:
        if workers is None:
            workers = default_workers()
        if workers <= 1 or len(items) < min_items or "fork" not in mp.get_all_start_methods():
            return [fn(it) for it in items]
        from concurrent.futures import ProcessPoolExecutor

        nch = min(len(items), workers * 8)
        bounds = np.linspace(0, len(items), nch + 1).astype(int)
        chunks = [items[bounds[i]:bounds[i + 1]] for i in range(nch)]
        out = []
        with ProcessPoolExecutor(max_workers=workers, mp_context=mp.get_context("fork"),
                                 initializer=_init_worker) as pool:
            for res in pool.map(_chunk, chunks):
                out.extend(res)
        return out
    finally:
        STATE.clear()
        _FN = None
