cd $GRAFT_REPO_ROOT
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 4
for P in 320 0 128 640; do
XDG_MF_PCOL=$P python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('PCOL=$P', json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual','factor_GB','setup_s')}))" | tee -a gpurun_out/r2_mf_pcol_sweep.jsonl
done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mf_ --csv --log-file gpurun_out/r2_mf_merged_launches_d.csv python tools/mf_levels.py native 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_merged_rows.json
python tools/launch_summary.py gpurun_out/r2_mf_merged_launches_d.csv | head
