cd $GRAFT_REPO_ROOT
# CPU job in the background (the host cores are otherwise idle during the GPU runs)
(timeout 3300 python tools/time_oracle_cfg2.py gpurun_out/oracle_cfg2_timing_box_gmres.json gmres:5 > gpurun_out/oracle_cfg2_timing_box_gmres.log 2>&1; echo "oracle gmres timing exit $?" >> gpurun_out/oracle_cfg2_timing_box_gmres.log) &
OR=$!
bash tools/_run13.sh 2>&1 | tee gpurun_out/r2_run13.txt
bash tools/sanitize.sh gpurun_out memcheck racecheck synccheck
cat gpurun_out/sanitize_summary.txt
for t in memcheck racecheck synccheck; do echo "== $t"; grep -c "ERROR SUMMARY\|error" gpurun_out/sanitize_$t.log; tail -n 3 gpurun_out/sanitize_$t.log; done
CELLS=96 timeout 1200 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed.jsonl; tail -n 2 gpurun_out/r2_cfg4_96cubed.jsonl | cut -c1-600
timeout 900 python tools/dist_lowfactor_memory.py cfg4 2>&1 | grep "^{" > gpurun_out/r2_dist_lowfactor_cfg4.jsonl; cat gpurun_out/r2_dist_lowfactor_cfg4.jsonl | cut -c1-400
wait $OR
tail -n 2 gpurun_out/oracle_cfg2_timing_box_gmres.log | cut -c1-800
