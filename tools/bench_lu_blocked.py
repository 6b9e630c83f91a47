"""Time the batched dense LU of Schwarz-like batches: unblocked batched
getrf (MAGMA) vs the blocked form (direct.lu_factor_blocked) per panel width.

    python tools/bench_lu_blocked.py [b n] ...   (default: cfg4 / cfg2 sizes)
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_02431_b200.direct import _lu_factor_unblocked, lu_factor_blocked  # noqa: E402

args = [int(a) for a in sys.argv[1:]] or [1100, 896, 340, 1920]
for b, n in zip(args[0::2], args[1::2]):
    A = torch.randn(b, n, n, dtype=torch.float64, device="cuda")
    A += n * torch.eye(n, dtype=torch.float64, device="cuda")
    row = {"batch": b, "n": n}
    for name, fn in [("unblocked", lambda: _lu_factor_unblocked(A))] + [
            (f"blocked{nb}", (lambda nb=nb: lu_factor_blocked(A, nb))) for nb in (64, 128, 256)]:
        fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        row[name + "_s"] = round(time.perf_counter() - t, 4)
    row["tflops_best"] = round(2 / 3 * n ** 3 * b / min(
        v for k, v in row.items() if k.endswith("_s")) / 1e12, 2)
    print(json.dumps(row), flush=True)
    del A
    torch.cuda.empty_cache()
