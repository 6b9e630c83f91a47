cd $GRAFT_REPO_ROOT
# session 5, call 9: the complete suite as the driver runs it (reference installed in baseline/_ref), with durations
( time python -m pytest tests/ -x -q -m gpu --durations=25 ) > gpurun_out/r2_gpu_tests_final2.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final2.txt
tail -n 45 gpurun_out/r2_gpu_tests_final2.txt | cut -c1-160
for leaf in 100 200 400 800; do
echo "== omg cfg2 XDG_MF_LEAF_MULTI=$leaf (cold, then 150 it steady)"
XDG_MF_LEAF_MULTI=$leaf python tools/profile_solve.py tests/golden/large/cfg2.npz omg 2>&1 | tail -n 1
XDG_MF_LEAF_MULTI=$leaf python tools/profile_solve.py tests/golden/large/cfg2.npz omg 150 --steady 2>&1 | tail -n 1
done | tee gpurun_out/r2_omg_mf_leaf_sweep.txt
python bench.py --steps 10 --warmup 3 --no-solve > gpurun_out/r2_bench_chunks12.json 2> gpurun_out/r2_bench_chunks12.err
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench_chunks12.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['e2e']['path'][:80])"
