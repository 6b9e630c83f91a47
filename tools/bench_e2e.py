"""Time HostStreamSpMV (host x -> device SpMV -> host y, overlapped) on the
BASELINE cfg3 operator for several chunk counts; also the raw pinned H2D /
D2H copy rates alone and concurrent.

    python tools/bench_e2e.py [n] [chunks ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.device import HostStreamSpMV  # noqa: E402
from paper_2003_02431_b200.synthetic import cfg3_slab_device  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
chunk_list = [int(a) for a in sys.argv[2:]] or [4, 8, 16, 32, 64]
s = cfg3_slab_device(n)
D = s["D"]
L = D.nbr * D.N
B = D.algorithmic_bytes()
xh = torch.randn(L, dtype=torch.float64).pin_memory()
yh = torch.empty(L, dtype=torch.float64).pin_memory()
xd = torch.empty(L, dtype=torch.float64, device="cuda")


def timed(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


out = {"bytes_per_vector": 8 * L}
out["h2d_ms"] = timed(lambda: xd.copy_(xh, non_blocking=True))
out["d2h_ms"] = timed(lambda: yh.copy_(xd, non_blocking=True))
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
xd2 = torch.empty_like(xd)


def duplex():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        xd.copy_(xh, non_blocking=True)
    with torch.cuda.stream(s2):
        yh.copy_(xd2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


out["duplex_ms"] = timed(duplex)
out["duplex_floor_GBs"] = B / out["duplex_ms"] / 1e6
for c in chunk_list:
    hs = HostStreamSpMV(D, chunks=c)

    def step():
        hs(xh, yh, sync=False)

    ms = timed(lambda: (step(), hs.wait()))
    out[f"chunks{c}_ms"] = ms
    out[f"chunks{c}_GBs"] = B / ms / 1e6
    # host-synchronous products (BlockSparseMatrix.matvec on pinned vectors,
    # the bench's e2e): the pipeline fills and drains inside every call
    import time as _t

    for _ in range(2):
        hs(xh, yh, sync=True)
    t0 = _t.perf_counter()
    for _ in range(10):
        hs(xh, yh, sync=True)
    out[f"chunks{c}_sync_GBs"] = B / ((_t.perf_counter() - t0) / 10) / 1e9
    # back-to-back products (one wait after K steps)
    for _ in range(2):
        step()
    hs.wait()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        step()
    hs.wait()
    b.record()
    b.synchronize()
    ms = a.elapsed_time(b) / 10
    out[f"chunks{c}_overlapped_GBs"] = B / ms / 1e6
print(json.dumps(out))
