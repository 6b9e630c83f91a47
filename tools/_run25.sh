cd $GRAFT_REPO_ROOT
# session 5, call 10: multifrontal Schwarz setup at cfg4 size (4,400 systems) after the host-side vectorisation
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py tests/test_pmg_gpu.py -q --timeout 2400 2>&1 | tail -n 3
CELLS=96 PROFILE_SORT=tottime PROFILE_LINES=40 timeout 1500 python tools/profile_setup_solve.py cfg4-native omg 2>&1 | grep -v Warning > gpurun_out/r2_cfg4_sparse_setup_prof.txt
head -n 56 gpurun_out/r2_cfg4_sparse_setup_prof.txt | cut -c1-170
CELLS=96 timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_auto_v2.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_auto_v2.jsonl | cut -c1-700
python tools/profile_solve.py tests/golden/large/cfg2.npz omg 2>&1 | tail -n 1
