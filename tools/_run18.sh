cd $GRAFT_REPO_ROOT
# session 5, call 3: low-order mode sweep (dense vs multifrontal Schwarz blocks), flat rm_step A/B, self-check
python -m pytest tests/test_selfcheck_gpu.py tests/test_large_solve_gpu.py -q --timeout 2400 -k "selfcheck or poison or backward_error" 2>&1 | tail -n 5
for mode in dense sparse; do
for case in tests/golden/large/cfg2.npz tests/golden/large/s16p3.npz tests/golden/sphere8p3.npz tests/golden/large/cfg4_16.npz tests/golden/cfg1.npz; do
echo "== omg $case XDG_LOW_ORDER=$mode (cold solve incl. lazy setup, then steady)"
XDG_LOW_ORDER=$mode python tools/profile_solve.py $case omg 2>&1 | tail -n 1
XDG_LOW_ORDER=$mode python tools/profile_solve.py $case omg --steady 2>&1 | tail -n 1
done; done | tee gpurun_out/r2_omg_loworder_full.txt
XDG_LOW_ORDER=sparse python -m pytest tests/test_pmg_gpu.py tests/test_solvers_gpu.py tests/test_large_gpu.py tests/test_omg_graph_gpu.py -q --timeout 2400 2>&1 | tail -n 6
for rep in 1 2 3; do
for flat in 0 1; do
for case in tests/golden/cfg1.npz tests/golden/sphere8p3.npz tests/golden/large/s16p3.npz; do
echo "== omg $case XDG_OMG_FLAT=$flat rep $rep"
XDG_OMG_FLAT=$flat python tools/profile_solve.py $case omg --steady 2>&1 | tail -n 1
done; done; done | tee gpurun_out/r2_omg_flat_ab.txt
