export HC_BENCH_NO_CLOCKS=1
timeout 900 python -m pytest tests/test_decoder_gpu.py tests/test_end_to_end_gpu.py -x -q 2>&1 | tail -2
for W in cfg4 cfg3 cfg5; do
timeout 600 python bench.py --workload $W --steps 300 --warmup 5 --no-cpu-baseline --secondary none > gpurun_out/pe_${W}.json 2> gpurun_out/pe_${W}.err; echo $W $?
done
