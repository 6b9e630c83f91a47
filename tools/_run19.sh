cd $GRAFT_REPO_ROOT
XDG_LOW_ORDER=sparse python tools/profile_setup_solve.py tests/golden/large/cfg2.npz omg 2>&1 | grep -v Warning | head -n 70 > gpurun_out/r2_omg_sparse_setup_prof.txt
head -n 60 gpurun_out/r2_omg_sparse_setup_prof.txt | cut -c1-180
for flat in 0 1 0 1; do
for case in tests/golden/cfg1.npz tests/golden/sphere8p3.npz; do
echo "== omg $case XDG_OMG_FLAT=$flat"
XDG_OMG_FLAT=$flat python tools/profile_solve.py $case omg --steady --repeat=6 2>&1 | tail -n 1
done; done | tee gpurun_out/r2_omg_flat_ab2.txt
