"""The graph-captured gmres_pmg_solve (restart cycles and Arnoldi steps as
nested WHILE nodes; device-side Givens / back substitution with the host
driver's rounding: xdg_driver.cu gmres_solve_graph) against the host-loop
driver (XDG_GMRES_GRAPH=0): identical iteration counts, residual histories
and solutions, bit for bit -- incl. the register-resident MGS kernel
(n >= 32,768: the 16^3 p=3 hierarchy) and restarts."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT, golden_path

pytestmark = pytest.mark.gpu

CODE = r"""
import hashlib, json, sys
import numpy as np
from conftest import golden_path
from paper_2003_02431_b200.hierarchy import load_hierarchy
from paper_2003_02431_b200.solvers import SolverConfig, gmres_pmg_solve
case, restart, tol, maxit = sys.argv[1], int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
z = np.load(golden_path(case))
meta = json.loads(bytes(z["meta"]).decode())
h = load_hierarchy(z)
lv = h.level(1)
cfg = dict(meta["gmres"], tolerance=tol, gmres_restart=restart, max_iterations=maxit)
for _ in range(2):
    x, r = gmres_pmg_solve(lv.matrix, np.asarray(lv.rhs), SolverConfig(**cfg), dim=meta["dim"])
print(json.dumps([r.iterations, r.converged, hashlib.sha1(np.asarray(x).tobytes()).hexdigest(),
                  hashlib.sha1(np.asarray(r.residual_history).tobytes()).hexdigest(),
                  r.time_iterations]))
"""


def _run(case, restart, tol, maxit, graph):
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, XDG_GMRES_GRAPH=graph, PYTHONPATH=os.pathsep.join([here, ROOT]))
    p = subprocess.run([sys.executable, "-c", CODE, case, str(restart), str(tol), str(maxit)],
                       env=env, capture_output=True, text=True, timeout=900, cwd=here)
    assert p.returncode == 0, p.stderr[-3000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("case,restart,tol,maxit", [
    ("bench4", 50, 1e-10, 3000), ("cfg1", 50, 1e-10, 3000), ("cfg1", 7, 1e-8, 400),
    ("sphere8p3", 50, 1e-10, 4000), ("large/s16p3", 50, 1e-8, 300)])
def test_graph_gmres_bit_identical_to_host_driver(case, restart, tol, maxit):
    if not os.path.exists(golden_path(case)):
        pytest.fail(f"fixture {case} missing")
    g = _run(case, restart, tol, maxit, "1")
    h = _run(case, restart, tol, maxit, "0")
    print(f"{case} m={restart}: graph {g[0]} it {g[4]:.3f}s | host {h[0]} it {h[4]:.3f}s")
    assert g[:4] == h[:4]
