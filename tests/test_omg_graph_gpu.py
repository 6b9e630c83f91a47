"""The graph-captured ortho_mg_solve (one CUDA graph, device-side RM
decisions and loop conditions: xdg_driver.cu omg_solve_graph) against the
host-decision driver (XDG_OMG_GRAPH=0): identical iteration counts,
residual histories and solutions, bit for bit (same kernels, same grids,
same arithmetic), on every fixture hierarchy incl. RM restarts (small
rm_max_columns) and a 4-level hierarchy."""
import hashlib
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, golden_path

pytestmark = pytest.mark.gpu

CODE = r"""
import hashlib, json, sys, time
import numpy as np
from conftest import golden_path
from paper_2003_02431_b200.hierarchy import load_hierarchy
from paper_2003_02431_b200.solvers import SolverConfig, ortho_mg_solve
case, cols, tol = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
z = np.load(golden_path(case))
meta = json.loads(bytes(z["meta"]).decode())
h = load_hierarchy(z)
cfg = dict(meta["omg"], tolerance=tol, rm_max_columns=cols)
x, r = ortho_mg_solve(h, np.asarray(h.level(1).rhs), None, SolverConfig(**cfg), 1)
x, r = ortho_mg_solve(h, np.asarray(h.level(1).rhs), None, SolverConfig(**cfg), 1)
print(json.dumps([r.iterations, r.converged, hashlib.sha1(np.asarray(x).tobytes()).hexdigest(),
                  hashlib.sha1(np.asarray(r.residual_history).tobytes()).hexdigest(),
                  r.time_iterations]))
"""


def _run(case, cols, tol, graph):
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, XDG_OMG_GRAPH=graph, PYTHONPATH=os.pathsep.join([here, ROOT]))
    p = subprocess.run([sys.executable, "-c", CODE, case, str(cols), str(tol)], env=env,
                       capture_output=True, text=True, timeout=900, cwd=here)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case,cols,tol", [("bench4", 200, 1e-10), ("cfg1", 200, 1e-10),
                                           ("cfg1", 7, 1e-8), ("sphere8p3", 800, 1e-10),
                                           ("cfg4_8", 200, 1e-8)])
def test_graph_omg_bit_identical_to_host_driver(case, cols, tol):
    if not os.path.exists(golden_path(case)):
        pytest.fail(f"fixture {case} missing")
    g = _run(case, cols, tol, "1")
    h = _run(case, cols, tol, "0")
    print(f"{case} cols={cols}: graph {g[0]} it {g[4]:.3f}s | host {h[0]} it {h[4]:.3f}s")
    assert g[:4] == h[:4]
