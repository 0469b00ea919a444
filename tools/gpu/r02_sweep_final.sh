bash tools/sweep_bench.sh
( time timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err ) 2> gpurun_out/final_bench.time
( time timeout 900 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err ) 2> gpurun_out/final_ref.time
tail -n 3 gpurun_out/final_bench.time gpurun_out/final_ref.time
