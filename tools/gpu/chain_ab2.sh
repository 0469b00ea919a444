timeout 900 python -m pytest tests/test_decoder_gpu.py -x -q 2>&1 | tail -1
run() { # tag lib workload
  HC_CHAIN_TRACE=1 HCB200_LIB=$2 HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload $3 --steps 300 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/ab_$1.json 2> gpurun_out/ab_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/ab_$1.json').read().strip().splitlines()[-1]);print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['retrieval']['landing_stall_ms_total'],2))"
  grep hc_chain_trace gpurun_out/ab_$1.err | grep -E "decide|fire_select|schedule|gathers|joins|main K4" | tr '\n' ' '; echo
}
NEW=paper_2601_13684_b200/libhcb200.so; OLD=paper_2601_13684_b200/libhcb200_old.so
for w in cfg2 cfg4; do
  run ${w}_old $OLD $w
  run ${w}_new $NEW $w
done
