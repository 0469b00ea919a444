export HC_BENCH_NO_CLOCKS=1 HC_NO_READ_PROBE=1
for W in cfg5 cfg3 cfg4; do
  B="python bench.py --workload $W --steps 16 --warmup 3 --no-cpu-baseline --secondary none"
  timeout 1500 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_$W.csv $B > gpurun_out/ncu_lf_$W.log 2>&1
  tail -1 gpurun_out/ncu_lf_$W.log
done
# one K4 + post kernels with --set full at cfg3 (final code)
B="python bench.py --workload cfg3 --steps 16 --warmup 3 --no-cpu-baseline --secondary none"
timeout 1500 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:attn_tiles_kernel -s 4 -c 1 -o gpurun_out/r02f_k4_cfg3 -f $B > gpurun_out/ncu_k4f.log 2>&1
tail -1 gpurun_out/ncu_k4f.log
