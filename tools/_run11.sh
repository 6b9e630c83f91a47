cd $GRAFT_REPO_ROOT
python -m pytest tests/test_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 4
python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual','factor_GB','setup_s')}))" | tee -a gpurun_out/r2_mf_pipe.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mf_ --csv --log-file gpurun_out/r2_mf_merged_launches_e.csv python tools/mf_levels.py native 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_merged_rows.json
python tools/mf_levels_pair.py gpurun_out/r2_mf_merged_rows.json gpurun_out/r2_mf_merged_launches_e.csv > gpurun_out/r2_mf_levels_merged_e.txt
cat gpurun_out/r2_mf_levels_merged_e.txt
