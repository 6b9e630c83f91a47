cd $GRAFT_REPO_ROOT
# session 5, call 15: multifrontal row-kernel launch bounds / loads in flight with the PDL chain (variants built by tools/build_mf_variants.sh)
for v in default minb4_u8 minb2_u8 minb3_u6 minb3_u12 minb4_u6 minb2_u12 minb2_u16; do
lib=paper_2003_02431_b200/libxdg_b200.so
[ $v != default ] && lib=variants/lib_$v.so
echo "== $v"
XDG_LIB=$PWD/$lib python tools/bench_mf.py tests/golden/large/cfg2.npz 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('solve_ms','min_ms','GBs','rel_residual') if k in d}))"
done | tee gpurun_out/r2_mf_variants.txt
