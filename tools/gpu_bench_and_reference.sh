timeout 1500 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo bench_rc=$?; tail -c 2500 gpurun_out/final_bench.json
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo ref_rc=$?; tail -c 600 gpurun_out/final_ref.json
