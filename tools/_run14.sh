cd $GRAFT_REPO_ROOT
python -m pytest tests -m gpu -q --timeout 2400 > gpurun_out/r2_gpu_tests_final.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final.txt
tail -n 8 gpurun_out/r2_gpu_tests_final.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -n 1 gpurun_out/r2_smoke.txt
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_bench_reference.json 2> gpurun_out/r2_bench_reference.err
echo "reference arm exit $?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
echo "bench exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/ncu_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:spmv_warp_rows --launch-skip 3 --launch-count 1 -o gpurun_out/r2_spmv_full -f python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/ncu_spmv.log 2>&1
ls -la gpurun_out/*.ncu-rep
