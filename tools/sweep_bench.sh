# Round bench lines of every workload (profiles/r02_bench_<cfg>.json; the default
# command's line is profiles/r02_bench_default.json) and the policies at cfg3.
set -u
for w in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 300 --warmup 5 --secondary none \
    > gpurun_out/sweep_$w.json 2> gpurun_out/sweep_$w.err
done
timeout 900 python bench.py --workload cfg4 --start-step 8192 --steps 300 --warmup 5 --secondary none \
  --no-cpu-baseline > gpurun_out/sweep_cfg4_t8k.json 2> gpurun_out/sweep_cfg4_t8k.err
for pol in full static_topk sink_window; do
  timeout 900 python bench.py --workload cfg3 --policy $pol --steps 100 --warmup 5 --secondary none \
    --no-cpu-baseline > gpurun_out/sweep_cfg3_$pol.json 2> gpurun_out/sweep_cfg3_$pol.err
done
for f in gpurun_out/sweep_*.json; do echo "$f $(grep -o '"value": [0-9.]*' $f | head -2 | tr '\n' ' ')"; done
