"""B200-native (sm_100a) drop-in for the solver hot path of the XDG
multigrid reference `cutdg` (arXiv 2003.02431).

Modules mirror the reference's names: `blockmatrix`, `solvers`, `errors`,
`transfer` (galerkin_restrict), `bench` (solve_assembled dispatch).  The
compute runs in the in-tree C-ABI library libxdg_b200.so
(include/xdg_b200.h); there is no CPU fallback.
"""
__version__ = "0.1.0"
