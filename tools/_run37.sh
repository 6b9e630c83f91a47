cd $GRAFT_REPO_ROOT
# session 5, call 21: cfg2 GMRES-PMG iteration count (chaotic at the 1e-10 floor) vs the group-task split knobs
for mode in "2048 2.0" "1024 2.0" "1536 2.0" "3072 2.0" "4096 2.0" "2048 1.5" "2048 3.0" "2048 1000"; do
set -- $mode
echo "== XDG_MF_LONG=$1 XDG_MF_CTA_WAVES=$2"
XDG_MF_LONG=$1 XDG_MF_CTA_WAVES=$2 python tools/profile_solve.py tests/golden/large/cfg2.npz gmres 10000 2>&1 | tail -n 1
done | tee gpurun_out/r2_gmres_cfg2_split_counts.txt
