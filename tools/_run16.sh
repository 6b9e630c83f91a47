cd $GRAFT_REPO_ROOT
# session 5, call 1: everything that does not need the (regenerating) cfg2 / cfg4_16 / cfg5 p3-5 fixtures
python -m pytest tests -m gpu -q --timeout 2400 -k "not cfg4_16 and not cfg5_10_p3 and not cfg5_10_p4 and not cfg5_10_p5" > gpurun_out/r2_gpu_tests_s5a.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_s5a.txt
tail -n 12 gpurun_out/r2_gpu_tests_s5a.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -n 2 gpurun_out/r2_smoke.txt
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_bench_reference_s5a.json 2> gpurun_out/r2_bench_reference_s5a.err
echo "reference arm exit $?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_s5a.json 2> gpurun_out/r2_bench_s5a.err
echo "bench exit $?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/ncu_bench.log 2>&1
echo "ncu launches exit $?"
ncu --set full --clock-control none --import-source on -k regex:spmv_warp_rows --launch-skip 3 --launch-count 1 -o gpurun_out/r2_spmv_full -f python bench.py --steps 2 --warmup 3 --no-solve --no-cpu > gpurun_out/ncu_spmv.log 2>&1
echo "ncu full exit $?"
ls -la gpurun_out/*.ncu-rep
bash tools/sanitize.sh gpurun_out memcheck racecheck synccheck
cat gpurun_out/sanitize_summary.txt
for t in memcheck racecheck synccheck; do echo "== $t"; tail -n 3 gpurun_out/sanitize_$t.log; done
XDG_INV_RING=1 python -m pytest tests/test_pmg_gpu.py tests/test_solvers_gpu.py -q --timeout 2400 -x 2>&1 | tail -n 4
python tools/bench_e2e.py 128 8 12 16 24 2>&1 | tail -n 1 | tee gpurun_out/r2_e2e_chunks.json
