cd $GRAFT_REPO_ROOT
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py tests/test_pmg_gpu.py tests/test_solvers_gpu.py tests/test_large_solve_gpu.py -q --timeout 2400 2>&1 | tail -n 3
CELLS=96 timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_auto_v5.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_auto_v5.jsonl | cut -c1-700
python tools/profile_solve.py tests/golden/large/cfg2.npz omg 2>&1 | tail -n 1
