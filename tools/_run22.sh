cd $GRAFT_REPO_ROOT
# session 5, call 7: full GPU suite with every fixture, both bench arms; CPU oracle GMRES timing at full cfg2 in the background (host cores idle during GPU runs)
(timeout 3400 python tools/time_oracle_cfg2.py gpurun_out/oracle_cfg2_timing_box_gmres.json gmres:5 > gpurun_out/oracle_cfg2_timing_box_gmres.log 2>&1; echo "oracle gmres timing exit $?" >> gpurun_out/oracle_cfg2_timing_box_gmres.log) &
OR=$!
python -m pytest tests -m gpu -q --timeout 3000 > gpurun_out/r2_gpu_tests_final.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gpu_tests_final.txt
tail -n 12 gpurun_out/r2_gpu_tests_final.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.txt 2>&1; tail -n 1 gpurun_out/r2_smoke.txt
wait $OR
tail -n 2 gpurun_out/oracle_cfg2_timing_box_gmres.log | cut -c1-900
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2_bench_reference_final.json 2> gpurun_out/r2_bench_reference_final.err
echo "reference arm exit $?"
python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench_final.json 2> gpurun_out/r2_bench_final.err
echo "bench exit $?"
