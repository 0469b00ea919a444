timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/final_tests.log; tail -2 gpurun_out/final_tests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
( time timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err ) 2> gpurun_out/final_bench.time
( time timeout 900 python bench.py --workload cfg3 > gpurun_out/final_bench_cfg3.json 2> gpurun_out/final_bench_cfg3.err ) 2> gpurun_out/final_bench_cfg3.time
if [ "${HC_FINAL_REF:-0}" = 1 ]; then
( time timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err ) 2> gpurun_out/final_ref.time
fi
tail -n 3 gpurun_out/final_bench.time
