"""The reference's own unit tests for the hot path, run verbatim against
this package (test_blockmatrix.py, test_solvers.py).  The test
files come with the reference install (tools/install_reference.sh ->
baseline/_ref/cutdg_tests); tests/ref_alias_plugin.py binds cutdg.blockmatrix
/ cutdg.solvers / cutdg.errors to this package before they are collected.
Skipped when the reference is not installed."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

SUITE = os.path.join(ROOT, "baseline", "_ref", "cutdg_tests")

# reference tests that inspect reference-private internals rather than the
# API contract (none so far); each entry says why
DESELECT: dict = {}


@pytest.mark.parametrize("fname", ["test_blockmatrix.py", "test_solvers.py"])
def test_reference_suite_against_package(fname):
    path = os.path.join(SUITE, fname)
    if not os.path.exists(path):
        pytest.skip("reference not installed (tools/install_reference.sh)")
    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([here, ROOT]),
               PYTHONDONTWRITEBYTECODE="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider",
           "-p", "ref_alias_plugin", "--rootdir", SUITE, path]
    for t, why in DESELECT.items():
        cmd += ["--deselect", f"{path}::{t}"]
    p = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=3000, cwd=SUITE)
    print(p.stdout[-4000:])
    assert p.returncode == 0, p.stdout[-6000:] + p.stderr[-2000:]
