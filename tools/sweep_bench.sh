# Round-end bench lines of every workload (profiles/r01_bench_<cfg>.json) and the
# launch list of the exact default command (profiles/r01_launches_cfg3.md source).
set -u
python bench.py > gpurun_out/sweep_cfg3.json 2> gpurun_out/sweep_cfg3.err
for w in cfg1 cfg2 cfg4 cfg5; do
  python bench.py --workload $w --no-cpu-baseline > gpurun_out/sweep_$w.json 2> gpurun_out/sweep_$w.err
done
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg3.csv python bench.py > gpurun_out/ncu_l.log 2>&1
for w in cfg3 cfg1 cfg2 cfg4 cfg5; do echo "$w $(grep -o '"value": [0-9.]*' gpurun_out/sweep_$w.json | head -2 | tr '\n' ' ') $(grep -o '"frac": [0-9.]*' gpurun_out/sweep_$w.json)"; done
