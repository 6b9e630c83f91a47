"""pytest plugin (test infrastructure): run the reference's own test bodies
(baseline/_ref/cutdg_tests, installed by tools/install_reference.sh) against
this package.  The reference's setup modules (mesh, basis, cut cells,
assembly, transfer) are imported first and stay the reference's; then the
hot-path modules the tests import by name -- cutdg.blockmatrix,
cutdg.solvers, cutdg.errors -- are replaced by this package's drop-ins, so
`from cutdg.solvers import gmres_pmg_solve` in a test body binds the B200
solver (import-compatible names, same semantics)."""
import importlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)

import cutdg  # noqa: E402

for m in ("errors", "blockmatrix", "solvers", "mesh", "basis", "levelset", "quadrature",
          "cutcells", "spaces", "agglomeration", "assembly", "transfer", "bench"):
    importlib.import_module(f"cutdg.{m}")

from paper_2003_02431_b200 import blockmatrix as _bm, errors as _er, solvers as _so  # noqa: E402

for name, mod in (("blockmatrix", _bm), ("solvers", _so), ("errors", _er)):
    sys.modules[f"cutdg.{name}"] = mod
    setattr(cutdg, name, mod)
