export HC_BENCH_NO_CLOCKS=1
timeout 900 python -m pytest tests/test_decoder_gpu.py -x -q 2>&1 | tail -2
for H in 1 2 4 8 0; do
HC_DEVDEC_HORIZON=$H timeout 600 python bench.py --workload cfg4 --steps 300 --warmup 5 --no-cpu-baseline --secondary none > gpurun_out/hz_cfg4_$H.json 2> gpurun_out/hz_cfg4_$H.err; echo H$H $?
done
HC_DEVDEC_HORIZON=2 timeout 600 python bench.py --workload cfg5 --steps 100 --warmup 5 --no-cpu-baseline --secondary none > gpurun_out/hz_cfg5_2.json 2> gpurun_out/hz_cfg5_2.err
