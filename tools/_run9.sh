cd $GRAFT_REPO_ROOT
python -m pytest tests/test_factor_gpu.py tests/test_multifrontal_gpu.py tests/test_dist_multifrontal_gpu.py -q --timeout 900 2>&1 | tail -n 6
XDG_MF_MERGE_SWEEP=0,1 python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 2 | tee gpurun_out/r2_mf_dmma_s4b.jsonl
