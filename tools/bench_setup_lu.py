"""Time batched dense LU + triangular inverses for Schwarz-like batches."""
import os
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2003_02431_b200.direct import triangular_inverses  # noqa: E402

torch.zeros(1).cuda()
dev = "cuda"


def batch(b, n):
    A = torch.randn(b, n, n, dtype=torch.float64, device=dev)
    A += n * torch.eye(n, dtype=torch.float64, device=dev)
    return A


def timeit(fn):
    torch.cuda.synchronize()
    t = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return time.perf_counter() - t


for lib in ("cusolver", "magma"):
    torch.backends.cuda.preferred_linalg_library(lib)
    for b, n in ((1, 1300), (8, 1300), (64, 1300), (16, 2500), (128, 512)):
        A = batch(b, n)
        torch.linalg.lu_factor_ex(A[:1])
        # silence MAGMA's advisory banner (stdout, C level)
        fd = os.dup(1)
        os.dup2(os.open(os.devnull, os.O_WRONLY), 1)
        try:
            t_lu = timeit(lambda: torch.linalg.lu_factor_ex(A))
            LU = torch.linalg.lu_factor_ex(A)[0]
            t_inv = timeit(lambda: triangular_inverses(LU))
        finally:
            os.dup2(fd, 1)
        print(f"{lib:8s} batch={b:4d} n={n:5d}: lu {t_lu * 1e3:8.1f} ms ({t_lu / b * 1e3:6.2f}/mat)"
              f"  inv {t_inv * 1e3:8.1f} ms", flush=True)
