for c in 1024 256 128; do
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg1 --steps 300 --warmup 5 --secondary none --chunk $c > gpurun_out/ch_$c.json 2> gpurun_out/ch_$c.err
python -c "import json;d=json.loads(open('gpurun_out/ch_$c.json').read().strip().splitlines()[-1]);print($c, d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'], d['parity']['within_tolerance'], d['phase_ms_per_step'])"
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg1 --steps 300 --warmup 5 --secondary none --chunk $c --l2 none > gpurun_out/chn_$c.json 2> gpurun_out/chn_$c.err
python -c "import json;d=json.loads(open('gpurun_out/chn_$c.json').read().strip().splitlines()[-1]);print('nofl', $c, d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms'])"
done
