timeout 900 python -m pytest tests/test_bench_contract.py -x -q 2>&1 | tail -2
HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload cfg1 --steps 300 --warmup 5 > gpurun_out/fl_cfg1.json 2> gpurun_out/fl_cfg1.err
python -c "import json;d=json.loads(open('gpurun_out/fl_cfg1.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['gpu_launches'], d['config']['l2'], d['roofline']['avg_launch_ms'], d['phase_ms_per_step'], d['timed_blocks_ms'])"
HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload cfg1 --steps 300 --warmup 5 --l2 none > gpurun_out/fl_cfg1n.json 2> gpurun_out/fl_cfg1n.err
python -c "import json;d=json.loads(open('gpurun_out/fl_cfg1n.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['config']['l2'])"
tail -3 gpurun_out/fl_cfg1.err
