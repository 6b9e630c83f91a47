cd $GRAFT_REPO_ROOT
# session 5, call 2: PDL chain for the multifrontal solve; full-size fixture tests; OMG low-order modes
XDG_MF_PDL=1 python -m pytest tests/test_multifrontal_gpu.py tests/test_gmres_graph_gpu.py tests/test_omg_graph_gpu.py -q --timeout 2400 -x 2>&1 | tail -n 4
for pdl in 0 1; do
echo "== XDG_MF_PDL=$pdl"
XDG_MF_PDL=$pdl python tools/bench_mf.py tests/golden/large/cfg2.npz 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual','setup_s') if k in d}))"
done | tee gpurun_out/r2_mf_pdl.txt
python -m pytest tests/test_large_gpu.py tests/test_large_solve_gpu.py tests/test_galerkin_gpu.py tests/test_configs_gpu.py -q --timeout 2400 -k "not cfg5_10_p3 and not cfg5_10_p4 and not cfg5_10_p5" > gpurun_out/r2_gpu_tests_s5b.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_s5b.txt
tail -n 8 gpurun_out/r2_gpu_tests_s5b.txt
for mode in "dense 0" "dense 1" "sparse 0"; do
set -- $mode
echo "== XDG_LOW_ORDER=$1 XDG_INV_RING=$2"
XDG_LOW_ORDER=$1 XDG_INV_RING=$2 python tools/profile_solve.py tests/golden/large/cfg2.npz omg 150 --steady 2>&1 | tail -n 1
done | tee gpurun_out/r2_omg_loworder_modes.txt
for pdl in 0 1; do
echo "== gmres XDG_MF_PDL=$pdl"
XDG_MF_PDL=$pdl python tools/profile_solve.py tests/golden/large/cfg2.npz gmres 300 --steady 2>&1 | tail -n 1
done | tee gpurun_out/r2_gmres_pdl.txt
XDG_OMG_FLAT=1 python -m pytest tests/test_omg_graph_gpu.py -q --timeout 2400 -x 2>&1 | tail -n 3
for flat in 0 1; do
for case in cfg1 sphere8p3; do
echo "== omg $case XDG_OMG_FLAT=$flat"
XDG_OMG_FLAT=$flat python tools/profile_solve.py tests/golden/$case.npz omg --steady 2>&1 | tail -n 1
done; done | tee gpurun_out/r2_omg_flat.txt
