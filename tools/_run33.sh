cd $GRAFT_REPO_ROOT
# session 5, call 16: rows per warp task x loads in flight of the whole-warp row path (variants: tools/build_mf_variants.sh mr)
for v in default mr3_mu8_minb2 mr3_mu12_minb2 mr3_mu6_minb2 mr3_mu10_minb2 mr3_mu8_minb3 mr5_mu6_minb2 mr6_mu6_minb2; do
lib=paper_2003_02431_b200/libxdg_b200.so
[ $v != default ] && lib=variants/lib_$v.so
echo "== $v"
XDG_LIB=$PWD/$lib python tools/bench_mf.py tests/golden/large/cfg2.npz 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual') if k in d}))"
done | tee gpurun_out/r2_mf_variants_mr3.txt
