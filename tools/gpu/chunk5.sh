for c in 1024 2048 1024 2048; do
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg5 --steps 100 --warmup 5 --secondary none --no-cpu-baseline --chunk $c > gpurun_out/ch5_$c.json 2> gpurun_out/ch5_$c.err
python -c "import json;d=json.loads(open('gpurun_out/ch5_$c.json').read().strip().splitlines()[-1]);print($c, round(d['value'],2), round(d['e2e']['value'],2), round(d['roofline']['avg_launch_ms'],3), d['phase_ms_per_step']['combine'], d['clocks']['sm_mhz'])"
done
