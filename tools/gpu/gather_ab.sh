run() { # tag env workload
  env $2 HC_CHAIN_TRACE=1 HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload $3 --steps 300 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/ga_$1.json 2> gpurun_out/ga_$1.err
  echo "$1 $(python -c "import json;d=json.loads(open('gpurun_out/ga_$1.json').read().strip().splitlines()[-1]);print(round(d['value'],1), round(d['e2e']['value'],1), round(d['retrieval']['landing_stall_ms_total'],2))") $(grep -E "gathers done|joins" gpurun_out/ga_$1.err | awk '{print $NF}' | tr '\n' ' ')"
}
for w in cfg2 cfg4; do
  run ${w}_40_256 X=1 $w
  run ${w}_148_256 HC_GATHER_CTAS=148 $w
  run ${w}_148_128 "HC_GATHER_CTAS=148 HC_GATHER_CHUNK=128" $w
  run ${w}_296_128 "HC_GATHER_CTAS=296 HC_GATHER_CHUNK=128" $w
done
run cfg5_40_256 X=1 cfg5
run cfg5_148_128 "HC_GATHER_CTAS=148 HC_GATHER_CHUNK=128" cfg5
