cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q --timeout 2400 -k "not cfg5_10_p5" > gpurun_out/r2_gpu_tests_s4c.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_s4c.txt
tail -n 25 gpurun_out/r2_gpu_tests_s4c.txt
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_s4c.json 2> gpurun_out/r2_bench_s4c.err
echo "bench exit $?"
