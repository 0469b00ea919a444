for c in 1024 512 2048 1024 512; do
HC_NO_READ_PROBE=1 timeout 900 python bench.py --workload cfg2 --steps 300 --warmup 5 --secondary none --no-cpu-baseline --chunk $c > gpurun_out/ch2_$c.json 2> gpurun_out/ch2_$c.err
python -c "import json;d=json.loads(open('gpurun_out/ch2_$c.json').read().strip().splitlines()[-1]);print($c, round(d['value'],1), round(d['e2e']['value'],1), round(d['roofline']['avg_launch_ms'],4), d['retrieval']['landing_stall_ms_total'])"
done
