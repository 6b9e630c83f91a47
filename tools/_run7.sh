cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none --import-source on -k regex:mf_merged --launch-skip 28 --launch-count 28 -o gpurun_out/r2_mf_merged_full -f python tools/mf_levels.py native 10 1 > /dev/null 2>&1
ls -la gpurun_out/*.ncu-rep
