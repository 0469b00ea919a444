export HC_BENCH_NO_CLOCKS=1
for B in 8 4 2 1; do
timeout 600 python bench.py --workload cfg5 --batch $B --steps 100 --warmup 5 --no-cpu-baseline --secondary none > gpurun_out/bs_cfg5_b$B.json 2> gpurun_out/bs_cfg5_b$B.err; echo B$B $?
done
for B in 4 2 1; do
timeout 600 python bench.py --workload cfg3 --batch $B --steps 200 --warmup 5 --no-cpu-baseline --secondary none > gpurun_out/bs_cfg3_b$B.json 2> gpurun_out/bs_cfg3_b$B.err; echo cfg3 B$B $?
done
