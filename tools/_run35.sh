cd $GRAFT_REPO_ROOT
# session 5, call 19: cfg2 GMRES-PMG solves (chaotic iteration count at the 1e-10 floor) for the fast multifrontal task shapes
for v in default mr2_mu8_minb3 mr2_mu8_minb2 mr4_mu8_minb2 mr4_mu12_minb2 mr3_mu10_minb2 mr3_mu6_minb2 mr3_mu12_minb2; do
lib=paper_2003_02431_b200/libxdg_b200.so
[ $v != default ] && lib=variants/lib_$v.so
echo "== $v"
XDG_LIB=$PWD/$lib python tools/profile_solve.py tests/golden/large/cfg2.npz gmres 2>&1 | tail -n 1
done | tee gpurun_out/r2_gmres_cfg2_variant_counts.txt
