"""Build SpMV launch-bound variants and time them (N=10 cfg3 128^3 operator,
N=20 cfg2 level-1 operator), plain and with the fused norm.

python tools/tune_spmv.py            # driver: builds + runs every variant
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
VARIANTS = [(3, 3, 0), (3, 3, 1), (3, 2, 1), (3, 4, 1)]


def build(small, large, flat20=0):
    out = f"/tmp/xdg_tune_{small}_{large}_{flat20}"
    os.makedirs(out, exist_ok=True)
    lib = os.path.join(out, "libxdg_b200.so")
    srcs = [os.path.join(ROOT, "paper_2003_02431_b200", "csrc", f) for f in
            sorted(os.listdir(os.path.join(ROOT, "paper_2003_02431_b200", "csrc")))
            if f.endswith(".cu")]
    subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-O3", "-std=c++17", "--shared", "-Xcompiler", "-fPIC", "--threads", "0",
                    f"-DXDG_SPMV_MINB_SMALL={small}", f"-DXDG_SPMV_MINB_LARGE={large}",
                    f"-DXDG_SPMV_FLAT20={flat20}",
                    "-I", os.path.join(ROOT, "include"), "-o", lib, *srcs], check=True)
    return lib


def measure():
    import numpy as np
    import torch

    sys.path.insert(0, ROOT)
    from paper_2003_02431_b200.hierarchy import load_hierarchy
    from paper_2003_02431_b200.synthetic import cfg3_slab_device

    res = {}
    cases = [("N10", cfg3_slab_device(128)["D"])]
    p = os.path.join(ROOT, "tests", "golden", "large", "cfg2.npz")
    if os.path.exists(p):
        cases.append(("N20", load_hierarchy(np.load(p), 1).level(1).matrix.device()))
    nrm = torch.zeros(1, dtype=torch.float64, device="cuda")
    for name, D in cases:
        x = torch.randn(D.nbc * D.N, dtype=torch.float64, device="cuda")
        y = torch.empty(D.nbr * D.N, dtype=torch.float64, device="cuda")
        for norm in (False, True):
            f = (lambda: D.spmv(x, y, norm_out=nrm)) if norm else (lambda: D.spmv(x, y))
            for _ in range(5):
                f()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                f()
            e.record()
            e.synchronize()
            ms = s.elapsed_time(e) / 20
            res[f"{name}{'_norm' if norm else ''}"] = round(D.algorithmic_bytes() / ms / 1e6, 1)
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    if "--measure" in sys.argv:
        measure()
    else:
        for sm, lg, f20 in VARIANTS:
            lib = build(sm, lg, f20)
            out = subprocess.run([sys.executable, __file__, "--measure"], capture_output=True,
                                 text=True, env=dict(os.environ, XDG_LIB=lib))
            print(f"MINB small={sm} large={lg} flat20={f20}:", out.stdout.strip().splitlines()[-1]
                  if out.stdout.strip() else out.stderr[-500:], flush=True)
