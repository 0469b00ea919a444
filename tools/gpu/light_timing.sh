timeout 900 python -m pytest tests/test_bench_contract.py tests/test_decoder_gpu.py -x -q 2>&1 | tail -2
for w in cfg1 cfg2 cfg3; do
  HC_HOST_PROF=1 timeout 600 python tools/host_cost.py --workload $w --steps 300 --warmup 5 > gpurun_out/lt_$w.json 2> gpurun_out/lt_$w.err
  echo "== $w"; grep "host_cost\|hc_host_prof" gpurun_out/lt_$w.err | tail -14
  python -c "import json;d=json.loads(open('gpurun_out/lt_$w.json').read().strip().splitlines()[-1]);print('$w', d['value'], d['e2e']['value'], d['gpu_launches'], d['roofline']['frac'], d['roofline']['avg_launch_ms'], d['phase_ms_per_step'])"
done
