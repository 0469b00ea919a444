export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tiles_kernel -s 10 -c 1 -o gpurun_out/k4_cfg3 -f $B > gpurun_out/ncu_k4.log 2>&1
tail -3 gpurun_out/ncu_k4.log
