"""Micro-benchmark: one-CTA vs whole-GPU triangular-inverse LU apply for a
single dense system of size n (decides direct.LARGE_MIN_N)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.direct import DeviceDirect  # noqa: E402

ctx = Context.get()
rng = np.random.default_rng(0)
for n in (128, 256, 512, 831, 1024, 1536, 2048, 4096, 5690):
    A = rng.standard_normal((n, n)) + n ** 0.5 * np.eye(n)
    b = torch.from_numpy(rng.standard_normal(n)).cuda()
    At = torch.from_numpy(A).cuda()
    row = [n]
    for _ in (0,):
        F = DeviceDirect(At, ctx)
        x = F.apply(b)
        for _ in range(5):
            F.apply(b, x)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(50):
            F.apply(b, x)
        e.record()
        e.synchronize()
        us = s.elapsed_time(e) * 1e3 / 50
        err = np.linalg.norm(x.cpu().numpy() - np.linalg.solve(A, b.cpu().numpy()))
        row += [round(us, 1), f"{err:.1e}"]
    print("n=%d  %.1f us (err %s)  %.1f GB/s" % (row[0], row[1], row[2], 8 * n * n / (row[1] * 1e3)), flush=True)
