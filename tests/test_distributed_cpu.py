"""Multi-rank host logic of the z-slab decomposition, on CPU with gloo
(world size 2 and 3): ghost lists, halo exchange, interior/boundary split,
and that the slab-local SpMV (oracle arithmetic on the local arrays) equals
the rows of the global reference product bit for bit."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, q):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import cfg3, spmv
        from paper_2003_02431_b200.distributed import HaloPlan, allreduce_sum, split_interior
        from paper_2003_02431_b200.synthetic import cfg3_slab_host

        rp_g, col_g, val_g, x_g = cfg3.build(n)
        y_g = spmv.bsr_spmv(rp_g, col_g, val_g, x_g)
        N = val_g.shape[1]
        h = cfg3_slab_host(n, rank, world)
        nloc = h["row1"] - h["row0"]
        starts = torch.tensor([h["row0"]], dtype=torch.int64)
        allst = [torch.zeros_like(starts) for _ in range(world)]
        dist.all_gather(allst, starts)
        row_starts = np.array([int(t) for t in allst] + [h["nbr_global"]])
        plan = HaloPlan(row_starts, h["ghosts"], rank, world, N, torch.device("cpu"))
        x_ext = torch.zeros((nloc + len(h["ghosts"])) * N, dtype=torch.float64)
        x_ext[: nloc * N] = torch.from_numpy(x_g[h["row0"] * N: h["row1"] * N])
        plan.exchange(x_ext)
        ghosts_ok = np.array_equal(
            x_ext[nloc * N:].numpy().reshape(-1, N), x_g.reshape(-1, N)[h["ghosts"]])
        val_loc = val_g[h["global_blocks"]]
        y_loc = spmv.bsr_spmv(h["row_ptr"], h["col"], val_loc, x_ext.numpy())
        y_ok = np.array_equal(y_loc, y_g[h["row0"] * N: h["row1"] * N])
        a, b = split_interior(h["row_ptr"], h["col"], nloc)
        rows_of = np.repeat(np.arange(nloc), np.diff(h["row_ptr"]))
        interior_ok = not np.any(h["col"][(rows_of >= a) & (rows_of < b)] >= nloc)
        s = allreduce_sum(torch.tensor([float(rank + 1)]))
        q.put((rank, ghosts_ok, y_ok, interior_ok, b > a or world == 1, float(s[0]),
               len(plan.sends), plan.nghost))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_halo_exchange_and_local_spmv(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 8, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ghosts_ok, y_ok, interior_ok, has_interior, s, nsend, nghost in res:
        assert ghosts_ok, rank
        assert y_ok, rank
        assert interior_ok and has_interior, rank
        assert s == world * (world + 1) / 2
        assert nghost > 0 and nsend >= 1


def test_halo_plan_single_rank_is_noop():
    sys.path.insert(0, ROOT)
    from paper_2003_02431_b200.distributed import HaloPlan

    plan = HaloPlan(np.array([0, 10]), np.zeros(0, np.int64), 0, 1, 4, torch.device("cpu"))
    assert plan.start(torch.zeros(40, dtype=torch.float64)) == []
