cd $GRAFT_REPO_ROOT
python -m pytest tests/test_factor_gpu.py tests/test_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 8
python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | tee gpurun_out/r2_mf_dmma_s4.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_mf_all_launches_b.csv python tools/mf_levels.py native 10 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2_mf_all_launches_b.csv > gpurun_out/r2_mf_setup_kernels_b.txt; head -12 gpurun_out/r2_mf_setup_kernels_b.txt
