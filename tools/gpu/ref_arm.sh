timeout 900 python -m pytest tests/test_end_to_end_gpu.py tests/test_bench_contract.py -x -q 2>&1 | tail -2
( time timeout 900 python bench.py --impl reference > gpurun_out/ref5.json 2> gpurun_out/ref5.err ) 2> gpurun_out/ref5.time
( time timeout 900 python bench.py --impl reference --workload cfg3 > gpurun_out/ref3.json 2> gpurun_out/ref3.err ) 2> gpurun_out/ref3.time
( time timeout 900 python bench.py --impl reference --workload cfg1 > gpurun_out/ref1.json 2> gpurun_out/ref1.err ) 2> gpurun_out/ref1.time
for f in ref5 ref3 ref1; do tail -n 3 gpurun_out/$f.time | head -1; python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d.get('extrapolation'), d['cpu_baseline'].get('sample'))"; done
