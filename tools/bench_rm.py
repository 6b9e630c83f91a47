"""Micro-benchmark of the residual-minimisation kernels at cfg2 size:
W^T w (xdg_gemv_t) and w -= W c, z -= Z c (xdg_gemv_update2)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.device import Context  # noqa: E402

ctx = Context.get()
n = 673220
for ncols in (50, 200, 400, 800):
    W = torch.randn(ncols, n, dtype=torch.float64, device="cuda")
    Z = torch.randn(ncols, n, dtype=torch.float64, device="cuda")
    w = torch.randn(n, dtype=torch.float64, device="cuda")
    z = torch.randn(n, dtype=torch.float64, device="cuda")
    c = torch.zeros(ncols, dtype=torch.float64, device="cuda")
    for name, fn, nbytes in (
            ("gemv_t", lambda: ctx.gemv_t(W, ncols, w, c), 8 * ncols * n + 8 * n),
            ("update2", lambda: ctx.gemv_update2(W, Z, ncols, c, w, z), 16 * ncols * n + 32 * n)):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        e.record()
        e.synchronize()
        ms = s.elapsed_time(e) / 10
        print(f"ncols={ncols:4d} {name:8s} {ms:8.3f} ms  {nbytes / ms / 1e6:7.0f} GB/s", flush=True)
    del W, Z
