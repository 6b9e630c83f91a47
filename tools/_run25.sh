cd $GRAFT_REPO_ROOT
# session 5, call 10: where the multifrontal Schwarz setup goes at cfg4 size (4,400 systems)
CELLS=96 PROFILE_SORT=tottime PROFILE_LINES=45 timeout 1500 python tools/profile_setup_solve.py cfg4-native omg 2>&1 | grep -v Warning > gpurun_out/r2_cfg4_sparse_setup_prof.txt
head -n 60 gpurun_out/r2_cfg4_sparse_setup_prof.txt | cut -c1-170
