timeout 900 python -m pytest tests/test_bench_contract.py -x -q 2>&1 | tail -2
for i in 1 2; do
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg4 --steps 300 --warmup 5 --secondary none > gpurun_out/st_cfg4_$i.json 2> gpurun_out/st_cfg4_$i.err
python -c "import json;d=json.loads(open('gpurun_out/st_cfg4_$i.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['timed_blocks_ms'], d['retrieval']['landing_stall_ms_total'], d['parity']['within_tolerance'], d['parity']['events_identical'], d['config']['settle_steps'])"
done
