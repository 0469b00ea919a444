for w in cfg2 cfg4; do
HC_CHAIN_TRACE=1 HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload $w --steps 300 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/ct_$w.json 2> gpurun_out/ct_$w.err
echo "== $w $(python -c "import json;d=json.loads(open('gpurun_out/ct_$w.json').read().strip().splitlines()[-1]);print(round(d['value'],1), d['retrieval']['landing_stall_ms_total'], d['phase_ms_per_step']['attention'])")"
grep hc_chain_trace gpurun_out/ct_$w.err | tail -12
done
