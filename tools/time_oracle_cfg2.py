"""Time the CPU oracle (oracle/solvers_np.py: the numpy/scipy restatement of
the reference solvers, pinned bit-exact against the reference's outputs by
tests/test_oracle.py) at full BASELINE config 2 on THIS host -- run on the
GPU box, so the cfg2 solve rows of bench.py carry a CPU baseline measured
on the same machine.  A full oracle solve takes hours (like the
reference's), so, as for the reference (tests/golden/time_reference_cfg2.py),
1 and 3 iterations are timed (the first includes the lazy factorizations
inside the solve timer, solvers.py:696 / 778) and the solve is
extrapolated: first + (iterations - 1) x per-iteration.

    python tools/time_oracle_cfg2.py [out.json]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import solvers_np as so  # noqa: E402
from paper_2003_02431_b200.hierarchy import fixture_array  # noqa: E402


def main(out, only=None):
    z = np.load(os.path.join(ROOT, "tests", "golden", "large", "cfg2.npz"))
    meta = json.loads(bytes(z["meta"]).decode())

    class Z(dict):
        files = property(lambda self: list(self.keys()))

    zz = Z()
    for k in z.files:
        if k.endswith("__uniq"):
            base = k[: -len("__uniq")]
            zz[base] = fixture_array(z, base)
        elif not k.endswith("__idx"):
            zz[k] = z[k]
    import platform

    res = {"host": platform.node(), "cores": os.cpu_count(),
           "blas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default (all cores)"),
           "cpu": open("/proc/cpuinfo").read().split("model name")[1].split("\n")[0].strip(": ")
           if os.path.exists("/proc/cpuinfo") else None,
           "what": "oracle/solvers_np.py (reference-exact numpy/scipy restatement), "
                   "large/cfg2 fixture (the reference's own hierarchy)",
           "dofs_raw": meta["dofs_raw"]}
    runs = [(sv, it) for sv in ("omg", "gmres") for it in (1, 3)]
    if only:  # e.g. "gmres:3,omg:1": a subset (merge with an earlier file by hand)
        runs = [(a.split(":")[0], int(a.split(":")[1])) for a in only.split(",")]
    for solver, its in runs:
        for _ in (0,):
            cfg = dict(tolerance=1e-10, schwarz_target_dofs=2000, rm_max_columns=200,
                       coarse_cycle_iterations=2, gmres_restart=30)
            cfg.update(meta[solver])
            cfg["k_lo"] = int(cfg["k_lo"])
            cfg["max_iterations"] = its
            h = so.hierarchy_from_npz(zz, meta["dim"])  # fresh caches: setup inside
            b = np.asarray(zz["L1_rhs"], float)
            t0 = time.perf_counter()
            if solver == "omg":
                _, it, hist = so.omg(h, b, cfg)
            else:
                lv = h.levels[0]
                tm = {}
                _, it, hist = so.gmres(lv["M"], lv["rp"], lv["col"], lv["val"], b, cfg,
                                       meta["dim"], timing=tm)
                # one factorization (35 min of SuperLU at cfg2) serves both
                # entries: 1 and 3 iterations from the per-iteration times
                res["gmres_setup_s"] = tm["setup_s"]
                res["gmres_iter_s"] = tm["iter_s"]
                if len(tm["iter_s"]) >= 3:
                    res["gmres_1it_s"] = tm["setup_s"] + tm["iter_s"][0]
                    res["gmres_3it_s"] = tm["setup_s"] + sum(tm["iter_s"][:3])
                    res["gmres_3it_residual"] = float(hist[3])
                    print(json.dumps(res), flush=True)
                    continue
            res[f"{solver}_{its}it_s"] = time.perf_counter() - t0
            res[f"{solver}_{its}it_residual"] = float(hist[-1])
            print(json.dumps(res), flush=True)
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else
         os.path.join(ROOT, "tests", "golden", "oracle_cfg2_timing_box.json"),
         sys.argv[2] if len(sys.argv) > 2 else None)
