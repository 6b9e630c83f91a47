cd $GRAFT_REPO_ROOT
# session 5, call 8: cfg4 at full size with the new low-order selection (auto vs dense); per-level multifrontal table and a full ncu capture with the PDL chain
CELLS=96 timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_auto.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_auto.jsonl | cut -c1-700
CELLS=96 XDG_LOW_ORDER=dense timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_dense.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_dense.jsonl | cut -c1-700
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:mf_ --csv --log-file gpurun_out/r2_mf_pdl_launches.csv python tools/mf_levels.py tests/golden/large/cfg2.npz 10 1 2>/dev/null | grep "^\[" > gpurun_out/r2_mf_pdl_rows.json
python tools/mf_levels_pair.py gpurun_out/r2_mf_pdl_rows.json gpurun_out/r2_mf_pdl_launches.csv > gpurun_out/r2_mf_levels_pdl.txt
head -n 50 gpurun_out/r2_mf_levels_pdl.txt
ncu --set full --clock-control none --import-source on -k regex:mf_merged --launch-skip 28 --launch-count 28 -o gpurun_out/r2_mf_merged_pdl_full -f python tools/mf_levels.py tests/golden/large/cfg2.npz 10 1 > gpurun_out/ncu_mf_full.log 2>&1
ls -la gpurun_out/*.ncu-rep
for mode in "1 0" "0 0" "0 tree:4" "0 tree:8" "0 level:3"; do
set -- $mode
echo "== omg cfg2 150 it steady XDG_MF_MERGE=$1 XDG_MF_FUSE=$2"
XDG_MF_MERGE=$1 XDG_MF_FUSE=$2 python tools/profile_solve.py tests/golden/large/cfg2.npz omg 150 --steady 2>&1 | tail -n 1
done | tee gpurun_out/r2_omg_schwarz_mf_modes.txt
timeout 1200 python tools/dist_lowfactor_memory.py cfg4 2>&1 | grep "^{" > gpurun_out/r2_dist_lowfactor_cfg4.jsonl; cut -c1-500 gpurun_out/r2_dist_lowfactor_cfg4.jsonl
for p in 1 2 3 4 5; do
timeout 900 python tools/time_setup.py --cells 48 --degree $p --radius 0.5 --solve omg 2>&1 | grep "^{" | tail -n 1
done > gpurun_out/r2_cfg5_psweep_48cubed.jsonl
cut -c1-90 gpurun_out/r2_cfg5_psweep_48cubed.jsonl; python - <<'PY'
import json
for l in open("gpurun_out/r2_cfg5_psweep_48cubed.jsonl"):
    d = json.loads(l)
    o = d.get("omg", {})
    print(d["degree"], d["raw_dofs"], d["setup_s"], o.get("iterations"), o.get("solve_s"), o.get("dof_per_s"), o.get("converged"))
PY
