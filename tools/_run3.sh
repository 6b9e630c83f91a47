cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mf_ --csv --log-file gpurun_out/r2_mf_merged_launches.csv python tools/mf_levels.py native 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_merged_rows.json
python tools/mf_levels_pair.py gpurun_out/r2_mf_merged_rows.json gpurun_out/r2_mf_merged_launches.csv > gpurun_out/r2_mf_levels_merged.txt
cat gpurun_out/r2_mf_levels_merged.txt
