cd $GRAFT_REPO_ROOT
out=gpurun_out/r2_mf_group_sweep.jsonl
: > $out
for cfg in "default 2048 2" "default 4096 2" "default 2048 1000" "default 1024 2" "default 2048 3" "gw8 2048 2" "gw2 2048 2" "gw8 4096 1000"; do
set -- $cfg
lib=$1; L=$2; W=$3
if [ $lib = default ]; then unset XDG_LIB; else export XDG_LIB=$PWD/build/variants/libxdg_$lib.so; fi
echo "== lib=$lib LONG=$L WAVES=$W" | tee -a $out
XDG_MF_LONG=$L XDG_MF_CTA_WAVES=$W python tools/bench_mf.py native 10 1 2>&1 | grep -v Warning | tail -n 1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({k:d[k] for k in ('lib','solve_ms','min_ms','GBs','setup_s')}))" | tee -a $out
done
