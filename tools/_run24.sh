cd $GRAFT_REPO_ROOT
# session 5, call 9: the complete suite as the driver runs it (reference installed in baseline/_ref), with durations
( time python -m pytest tests/ -x -q -m gpu --durations=25 ) > gpurun_out/r2_gpu_tests_final2.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final2.txt
tail -n 45 gpurun_out/r2_gpu_tests_final2.txt | cut -c1-160
