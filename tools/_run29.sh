cd $GRAFT_REPO_ROOT
for r in 1 2; do python tools/check_determinism.py 48 3 2>&1 | tail -n 1; done | tee gpurun_out/r2_determinism_cfg5_p3.txt
