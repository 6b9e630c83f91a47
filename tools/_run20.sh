cd $GRAFT_REPO_ROOT
# session 5, call 5: single-upload batched_factor, vectorised multifrontal plan, Schwarz low-order auto selection
python -m pytest tests/test_factor_gpu.py tests/test_multifrontal_gpu.py tests/test_pmg_gpu.py tests/test_solvers_gpu.py tests/test_large_gpu.py tests/test_large_solve_gpu.py tests/test_dist_multifrontal_gpu.py -q --timeout 2400 2>&1 | tail -n 6
python tools/profile_setup_solve.py tests/golden/large/cfg2.npz omg 2>&1 | grep -v Warning | head -n 40 > gpurun_out/r2_omg_auto_setup_prof.txt
head -n 30 gpurun_out/r2_omg_auto_setup_prof.txt | cut -c1-160
for case in tests/golden/large/cfg2.npz tests/golden/large/s16p3.npz; do
echo "== omg $case auto (cold, steady)"
python tools/profile_solve.py $case omg 2>&1 | tail -n 1
python tools/profile_solve.py $case omg --steady 2>&1 | tail -n 1
done | tee gpurun_out/r2_omg_auto.txt
python tools/profile_setup_solve.py tests/golden/large/cfg2.npz gmres 2>&1 | grep -v Warning | head -n 30 | cut -c1-160 > gpurun_out/r2_gmres_setup_prof.txt
head -n 12 gpurun_out/r2_gmres_setup_prof.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_s5c.json 2> gpurun_out/r2_bench_s5c.err
echo "bench exit $?"
