timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_bench_contract.py -x -q 2>&1 | tail -2
for w in cfg1; do
  HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload $w --steps 300 --warmup 5 > gpurun_out/sio_$w.json 2> gpurun_out/sio_$w.err
  python -c "import json;d=json.loads(open('gpurun_out/sio_$w.json').read().strip().splitlines()[-1]);print('$w', d['value'], d['e2e']['value'], d['gpu_launches'], d['parity']['within_tolerance'])"
  HC_HOST_PROF=1 HC_NO_READ_PROBE=1 timeout 600 python tools/host_cost.py --workload $w --steps 300 --warmup 5 > gpurun_out/lt_$w.json 2> gpurun_out/lt_$w.err
  grep "host_cost\|hc_host_prof" gpurun_out/lt_$w.err | tail -16
done
