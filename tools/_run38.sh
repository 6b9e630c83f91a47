cd $GRAFT_REPO_ROOT
# session 5, call 22: final state (group-task threshold 3 x 3,552 warp tasks)
( time python -m pytest tests/ -x -q -m gpu ) > gpurun_out/r2_gpu_tests_final5.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final5.txt
tail -n 8 gpurun_out/r2_gpu_tests_final5.txt | cut -c1-160
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -n 1 gpurun_out/r2_smoke.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_final4.json 2> gpurun_out/r2_bench_final4.err
echo "bench exit $?"
python -c "
import json
d = json.loads(open('gpurun_out/r2_bench_final4.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'], d['roofline']['frac'])
for r in d['solve']:
    print(r['case'], r['solver'], r.get('iterations'), r.get('solve_s'), r.get('dof_per_s'), r.get('setup_s'), r.get('loop_frac_of_hbm_peak'))
"
python tools/bench_mf.py tests/golden/large/cfg2.npz 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual') if k in d}))" | tee gpurun_out/r2_mf_final.txt
