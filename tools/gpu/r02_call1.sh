set -x
nproc; free -g | head -2; lscpu | grep -i "model name\|socket\|numa node(s)"
timeout 1200 python tools/selection_precision.py > gpurun_out/selprec.log 2>&1; echo selprec_rc=$?
timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline > gpurun_out/bench_fp32.json 2> gpurun_out/bench_fp32.err; echo b1=$?
timeout 300 python bench.py --steps 60 --warmup 5 --no-cpu-baseline --score-material fp16 > gpurun_out/bench_fp16.json 2> gpurun_out/bench_fp16.err; echo b2=$?
