# Round profile set for one workload (default cfg5): bench line, ncu launch list of
# the timed loop, ncu --set full of one K4 launch and of the post-attention kernels
# inside it (NVTX range "timed": calibration decodes in setup also launch K4).
W=${1:-cfg5}
R=${2:-r02}
export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload $W --steps 16 --warmup 3 --no-cpu-baseline --secondary none"
$B > gpurun_out/${R}_prof_b16_$W.json 2>&1 || exit 1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_launches_$W.csv $B > gpurun_out/ncu_l.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:attn_tiles_kernel -s 4 -c 1 -o gpurun_out/${R}_k4_$W -f $B > gpurun_out/ncu_k4.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"monitor_kernel|score_rows_kernel|combine_kernel|append_kernel" -s 8 -c 4 -o gpurun_out/${R}_post_$W -f $B > gpurun_out/ncu_post.log 2>&1
tail -2 gpurun_out/ncu_l.log gpurun_out/ncu_k4.log gpurun_out/ncu_post.log
