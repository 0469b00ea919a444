export HC_BENCH_NO_CLOCKS=1
B="python bench.py --workload cfg5 --layers 8 --steps 16 --warmup 3 --no-cpu-baseline --secondary none --roles fixed"
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:fire_select --clock-control none --csv --log-file gpurun_out/fs_a.csv $B > /dev/null 2>&1
HC_DEVDEC_NO_HOST_COPY=1 timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum -k regex:fire_select --clock-control none --csv --log-file gpurun_out/fs_b.csv $B > /dev/null 2>&1
timeout 600 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum -k regex:fire_select --clock-control none --csv --log-file gpurun_out/fs_c.csv $B --decisions host > /dev/null 2>&1
grep -h "gpu__time_duration" gpurun_out/fs_a.csv gpurun_out/fs_b.csv gpurun_out/fs_c.csv | awk -F'","' '{print $(NF)}'
