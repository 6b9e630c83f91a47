cd $GRAFT_REPO_ROOT
python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 > gpurun_out/r2_mf_merge_s4b.jsonl
cat gpurun_out/r2_mf_merge_s4b.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mf_all_launches.csv python tools/mf_levels.py native 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_merged_rows.json
python tools/mf_levels_pair.py gpurun_out/r2_mf_merged_rows.json gpurun_out/r2_mf_all_launches.csv > gpurun_out/r2_mf_levels_merged_b.txt
cat gpurun_out/r2_mf_levels_merged_b.txt
python tools/launch_summary.py gpurun_out/r2_mf_all_launches.csv > gpurun_out/r2_mf_setup_kernels.txt
cat gpurun_out/r2_mf_setup_kernels.txt
