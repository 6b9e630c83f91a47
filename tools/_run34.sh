cd $GRAFT_REPO_ROOT
# session 5, call 18: multifrontal row kernels with 3 rows per warp task, 2 resident CTAs per SM (adopted from the variant sweep)
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py tests/test_gmres_graph_gpu.py tests/test_omg_graph_gpu.py tests/test_pmg_gpu.py tests/test_solvers_gpu.py tests/test_large_solve_gpu.py tests/test_selfcheck_gpu.py -q --timeout 2400 2>&1 | tail -n 3
for w in 2.0 3.0 1.0; do
echo "== XDG_MF_CTA_WAVES=$w"
XDG_MF_CTA_WAVES=$w python tools/bench_mf.py tests/golden/large/cfg2.npz 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual') if k in d}))"
done | tee gpurun_out/r2_mf_mr3_waves.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_final2.json 2> gpurun_out/r2_bench_final2.err
echo "bench exit $?"
python -c "
import json
d = json.loads(open('gpurun_out/r2_bench_final2.json').read().strip().splitlines()[-1])
print(d['value'], d['e2e']['value'])
for r in d['solve']:
    print(r['case'], r['solver'], r.get('iterations'), r.get('solve_s'), r.get('dof_per_s'), r.get('setup_s'))
"
