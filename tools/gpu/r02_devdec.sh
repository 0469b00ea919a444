export HC_BENCH_NO_CLOCKS=1
timeout 900 python -m pytest tests/test_decoder_gpu.py -x -q 2>&1 | tail -3
for W in cfg4 cfg3 cfg5; do for D in device; do
timeout 600 python bench.py --workload $W --steps 300 --warmup 5 --no-cpu-baseline --secondary none --decisions $D > gpurun_out/dd_${W}_$D.json 2> gpurun_out/dd_${W}_$D.err; echo $W $D $?
done; done
timeout 600 python bench.py --workload cfg4 --steps 300 --warmup 5 --no-cpu-baseline --secondary none --start-step 8192 > gpurun_out/dd_cfg4_8k_device.json 2> gpurun_out/dd_cfg4_8k.err; echo 8k $?
