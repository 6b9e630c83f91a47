cd $GRAFT_REPO_ROOT
for L in 2048 4096 1024; do
XDG_MF_LONG=$L python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | tee -a gpurun_out/r2_mf_long_sweep.jsonl
done
python -m pytest tests/test_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 4
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mf_ --csv --log-file gpurun_out/r2_mf_merged_launches_c.csv python tools/mf_levels.py native 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_merged_rows.json
python tools/mf_levels_pair.py gpurun_out/r2_mf_merged_rows.json gpurun_out/r2_mf_merged_launches_c.csv > gpurun_out/r2_mf_levels_merged_c.txt
cat gpurun_out/r2_mf_levels_merged_c.txt
