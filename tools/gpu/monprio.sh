run() { # tag env workload extra
  env $2 HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload $3 --steps 200 --warmup 5 --secondary none --no-cpu-baseline $4 > gpurun_out/mp_$1.json 2> gpurun_out/mp_$1.err
  python -c "import json;d=json.loads(open('gpurun_out/mp_$1.json').read().strip().splitlines()[-1]);r=d['retrieval'];print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],4), r['landing_stall_ms_total'], d['phase_ms_per_step']['append'])"
}
for rep in 1 2; do
  for w in cfg3 cfg4 cfg5; do
    run ${w}_hi_$rep X=1 $w ""
    run ${w}_lo_$rep HC_MON_PRIO_LO=1 $w ""
  done
done
