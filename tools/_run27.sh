cd $GRAFT_REPO_ROOT
# session 5, call 12: final state -- the driver's commands, then cfg4 at full size
( time python -m pytest tests/ -x -q -m gpu ) > gpurun_out/r2_gpu_tests_final3.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final3.txt
tail -n 8 gpurun_out/r2_gpu_tests_final3.txt | cut -c1-160
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -n 1 gpurun_out/r2_smoke.txt
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_bench_reference_final.json 2> gpurun_out/r2_bench_reference_final.err
echo "reference arm exit $?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
echo "bench exit $?"
CELLS=96 timeout 1500 python tools/bench_cfg4.py omg 2>&1 | grep "^{" > gpurun_out/r2_cfg4_96cubed_auto_v4.jsonl; tail -n 1 gpurun_out/r2_cfg4_96cubed_auto_v4.jsonl | cut -c1-700
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches exit $?"
