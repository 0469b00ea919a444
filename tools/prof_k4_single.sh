# K4 DRAM traffic per launch with single-pass metrics (no kernel replay: the
# full set's memory save/restore is impractical with cfg5's 94 GB resident).
W=${1:-cfg5}
R=${2:-r02}
export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload $W --steps 16 --warmup 3 --no-cpu-baseline --secondary none"
timeout 1200 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:attn_tiles_kernel -s 4 -c 2 --csv --log-file gpurun_out/${R}_k4single_$W.csv $B > gpurun_out/ncu_k4single_$W.log 2>&1
tail -3 gpurun_out/ncu_k4single_$W.log
