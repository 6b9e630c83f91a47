"""cProfile of the multifrontal factorization setup (Multifrontal.__init__)
on a fixture's level operator (default: cfg2 level 1, m = 10 low modes --
the GMRES-PMG global low-order system).

    python tools/profile_mf_setup.py tests/golden/large/cfg2.npz [m] [level]
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.blockmatrix import BlockSparseMatrix, uniform_layout  # noqa: E402
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.device import Context  # noqa: E402
from paper_2003_02431_b200.factor import warmup  # noqa: E402
from paper_2003_02431_b200.hierarchy import fixture_array  # noqa: E402
from paper_2003_02431_b200.multifrontal import Multifrontal  # noqa: E402

path = sys.argv[1]
m = int(sys.argv[2]) if len(sys.argv) > 2 else 10
lam = int(sys.argv[3]) if len(sys.argv) > 3 else 1
z = np.load(path)
rp, col = z[f"L{lam}_row_ptr"], z[f"L{lam}_col"]
val = fixture_array(z, f"L{lam}_val")
N, nb = val.shape[1], len(rp) - 1
M = BlockSparseMatrix.from_bsr(rp, col, val, uniform_layout(nb, N), uniform_layout(nb, N))
ctx = Context.get()
D = M.device(ctx)
warmup(Context.get())
v = np.arange(nb, dtype=np.int64)
Multifrontal(ctx, rp, col, D.val_t, N, [v], m, v * N, v * m)  # warm (MAGMA, kernels)
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
mf = Multifrontal(ctx, rp, col, D.val_t, N, [v], m, v * N, v * m)
torch.cuda.synchronize()
pr.disable()
print(f"setup {time.perf_counter() - t0:.3f} s, phases {mf.times}")
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
