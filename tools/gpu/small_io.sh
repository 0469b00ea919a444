timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_bench_contract.py tests/test_end_to_end_gpu.py -x -q 2>&1 | tail -2
for w in cfg1 cfg2; do
  HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload $w --steps 300 --warmup 5 > gpurun_out/sio_$w.json 2> gpurun_out/sio_$w.err
  python -c "import json;d=json.loads(open('gpurun_out/sio_$w.json').read().strip().splitlines()[-1]);print('$w', d['value'], d['e2e'], d['gpu_launches'], d['parity'])"
done
