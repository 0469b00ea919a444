# Round profile set for one workload (default cfg3): bench line, ncu launch list of
# the timed region, ncu --set full of K4 and of the post-attention kernels.
W=${1:-cfg3}
export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload $W --steps 16 --warmup 3 --no-cpu-baseline"
$B > gpurun_out/prof_b16_$W.json 2>&1 || exit 1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_tiles_kernel -s 10 -c 1 -o gpurun_out/k4_$W -f $B > gpurun_out/ncu_k4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"monitor_kernel|score_rows_kernel|combine_kernel|append_kernel" -s 9 -c 4 -o gpurun_out/post_$W -f $B > gpurun_out/ncu_post.log 2>&1
ls -la gpurun_out
