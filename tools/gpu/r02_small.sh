export HC_BENCH_NO_CLOCKS=1
for W in cfg1 cfg2; do
timeout 600 python bench.py --workload $W --steps 300 --warmup 5 --secondary none > gpurun_out/sm_$W.json 2> gpurun_out/sm_$W.err; echo $W $?
done
bash tools/prof_k4_single.sh cfg5 r02
B="python bench.py --workload cfg5 --steps 16 --warmup 3 --no-cpu-baseline --secondary none"
timeout 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_cfg5_dd.csv $B > gpurun_out/ncu_l5.log 2>&1; echo l5 $?
