cd $GRAFT_REPO_ROOT
XDG_MF_MERGE_SWEEP=0,1 python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 4 > gpurun_out/r2_mf_merge_s4a.jsonl
cat gpurun_out/r2_mf_merge_s4a.jsonl
python -m pytest tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 8
