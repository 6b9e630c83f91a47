cd $GRAFT_REPO_ROOT
timeout 2400 python tools/time_oracle_cfg2.py gpurun_out/oracle_cfg2_timing_box.json > gpurun_out/oracle_cfg2_timing_box.log 2>&1
echo "oracle timing exit $?"
tail -n 2 gpurun_out/oracle_cfg2_timing_box.log | cut -c1-600
for tool in memcheck racecheck synccheck; do
  timeout 1500 bash tools/sanitize.sh $tool
  echo "$tool exit $?"
done
