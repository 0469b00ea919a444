for w in cfg1; do
 for nt in 0 1; do
  HC_HOST_PROF=1 HC_BENCH_NO_TIMING=$nt HC_NO_READ_PROBE=1 timeout 600 python tools/host_cost.py --workload $w --steps 300 --warmup 5 > gpurun_out/hc_$w.json 2> gpurun_out/hc_$w.err
  echo "== $w no_timing=$nt"; grep "host_cost\|hc_host_prof" gpurun_out/hc_$w.err
  python -c "import json;d=json.loads(open('gpurun_out/hc_$w.json').read().strip().splitlines()[-1]);print('$w', d['value'], d['e2e']['value'], d['gpu_launches'])"
 done
done
