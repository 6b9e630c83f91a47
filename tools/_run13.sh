cd $GRAFT_REPO_ROOT
python -m pytest tests/test_factor_gpu.py tests/test_large_solve_gpu.py tests/test_configs_gpu.py -q --timeout 2400 -k "factor or backward_error or cfg5_10_p3 or cfg5_10_p5" 2>&1 | tail -n 6
XDG_INV_RING=1 python -m pytest tests/test_pmg_gpu.py tests/test_solvers_gpu.py -q --timeout 2400 -x 2>&1 | tail -n 4
python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','rel_residual','setup_s','times')}))"
python tools/bench_e2e.py 128 8 12 16 24 2>&1 | tail -n 1 | tee gpurun_out/r2_e2e_chunks.json
for mode in "dense 0" "dense 1" "sparse 0"; do
set -- $mode
echo "== XDG_LOW_ORDER=$1 XDG_INV_RING=$2"
XDG_LOW_ORDER=$1 XDG_INV_RING=$2 python tools/profile_solve.py tests/golden/large/cfg2.npz omg 150 --steady 2>&1 | tail -n 1
done
