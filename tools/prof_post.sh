# ncu of the per-step post-attention kernels (score rows, monitor, combine) at cfg3
export HC_BENCH_NO_CLOCKS=1
B="python bench.py --steps 16 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/b16.json 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${1:-monitor_kernel|score_rows_kernel|combine_kernel}" -s 9 -c ${2:-3} -o gpurun_out/post_cfg3 -f $B > gpurun_out/ncu2.log 2>&1
