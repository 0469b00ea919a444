timeout 1500 python -m pytest tests/test_decoder_gpu.py tests/test_end_to_end_gpu.py tests/test_scale_parity_gpu.py tests/test_bench_contract.py -x -q 2>&1 | tail -2
run() { # tag env workload steps
  env $2 HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload $3 --steps $4 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/pf_$1.json 2> gpurun_out/pf_$1.err
  echo "$1 $(python -c "import json;d=json.loads(open('gpurun_out/pf_$1.json').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['e2e']['value'],1), round(d['retrieval']['landing_stall_ms_total'],2), d['parity'] and d['parity']['within_tolerance'])" 2>&1 | tail -1)"
}
for w in cfg2 cfg4; do
  run ${w}_off HC_PIVOT_FIRST=0 $w 300
  run ${w}_on X=1 $w 300
  run ${w}_off2 HC_PIVOT_FIRST=0 $w 300
  run ${w}_on2 X=1 $w 300
done
for w in cfg3 cfg5; do
  run ${w}_off HC_PIVOT_FIRST=0 $w 100
  run ${w}_on X=1 $w 100
done
