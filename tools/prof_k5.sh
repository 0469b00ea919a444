# ncu --set full of the two K5 passes (obs_score_kernel) of one prefill layer
W=${1:-cfg3}
export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload $W --steps 4 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:obs_score_kernel -s 4 -c 2 -o gpurun_out/k5_$W -f $B > gpurun_out/ncu_k5.log 2>&1
tail -2 gpurun_out/ncu_k5.log
