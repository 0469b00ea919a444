for a in "--steps 1 --warmup 3" "--steps 7 --warmup 3" "--gpus 1 --steps 10 --warmup 4"; do
  HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload cfg1 --secondary none $a > gpurun_out/odd.json 2> gpurun_out/odd.err; echo "rc=$? $a"
  python -c "import json;d=json.loads(open('gpurun_out/odd.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['steps'], d['parity'] and d['parity']['within_tolerance'])" || tail -5 gpurun_out/odd.err
done
HC_NO_READ_PROBE=1 timeout 600 python bench.py --workload cfg3 --layers 2 --secondary none --steps 5 --warmup 3 > gpurun_out/odd.json 2> gpurun_out/odd.err; echo "rc=$? cfg3 small"
python -c "import json;d=json.loads(open('gpurun_out/odd.json').read().strip().splitlines()[-1]);print(d['value'], d['e2e']['value'], d['parity'] and d['parity']['within_tolerance'])" || tail -5 gpurun_out/odd.err
