timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_end_to_end_gpu.py -x -q 2>&1 | tail -2
for i in 1 2; do
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg4 --steps 300 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/dc_cfg4_$i.json 2> gpurun_out/dc_cfg4_$i.err
python -c "import json;d=json.loads(open('gpurun_out/dc_cfg4_$i.json').read().strip().splitlines()[-1]);print('cfg4', round(d['value'],1), round(d['e2e']['value'],1), d['retrieval']['landing_stall_ms_total'], d['timed_blocks_ms'])"
done
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg2 --steps 300 --warmup 5 --secondary none --no-cpu-baseline > gpurun_out/dc_cfg2.json 2> gpurun_out/dc_cfg2.err
python -c "import json;d=json.loads(open('gpurun_out/dc_cfg2.json').read().strip().splitlines()[-1]);print('cfg2', round(d['value'],1), round(d['e2e']['value'],1), d['retrieval']['landing_stall_ms_total'])"
export HC_BENCH_NO_CLOCKS=1 HC_NO_READ_PROBE=1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dc_launches_cfg4.csv python bench.py --workload cfg4 --steps 16 --warmup 3 --no-cpu-baseline --secondary none > /dev/null 2>&1
grep -i "decide_kernel" gpurun_out/dc_launches_cfg4.csv | head -3 | cut -c1-300
