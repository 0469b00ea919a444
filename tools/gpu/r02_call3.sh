( time timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err ) 2> gpurun_out/bench_default.time
echo bench_rc=$?; free -g | head -2
( time timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/ref_default.json 2> gpurun_out/ref_default.err ) 2> gpurun_out/ref_default.time
echo ref_rc=$?
timeout 1200 python -m pytest tests/test_bench_contract.py -x -q -m gpu 2>&1 | tail -15
