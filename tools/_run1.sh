cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q --timeout 1500 -k "not cfg2 and not cfg5_10_p3 and not cfg5_10_p4 and not cfg5_10_p5 and not cfg4_16" > gpurun_out/r2_gpu_tests_s4b.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_s4b.txt
tail -n 25 gpurun_out/r2_gpu_tests_s4b.txt
