cd $GRAFT_REPO_ROOT
# session 5, call 11: vectorised extend-add grouping, flat ragged arrays, threaded dissection
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py tests/test_factor_gpu.py tests/test_pmg_gpu.py tests/test_solvers_gpu.py tests/test_large_solve_gpu.py tests/test_configs_gpu.py -q --timeout 2400 2>&1 | tail -n 4
CELLS=96 PROFILE_SORT=tottime PROFILE_LINES=30 timeout 1500 python tools/profile_setup_solve.py cfg4-native omg 2>&1 | grep -v Warning > gpurun_out/r2_cfg4_sparse_setup_prof_v2.txt
head -n 40 gpurun_out/r2_cfg4_sparse_setup_prof_v2.txt | cut -c1-170
CELLS=96 timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_auto_v3.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_auto_v3.jsonl | cut -c1-700
python tools/profile_solve.py tests/golden/large/cfg2.npz omg 2>&1 | tail -n 1
