( time python bench.py --steps 20 --warmup 5 ) > gpurun_out/bench_c3p6.json 2> gpurun_out/bench_c3p6.err
tail -3 gpurun_out/bench_c3p6.err
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/ref_c3p6.json 2> gpurun_out/ref_c3p6.err
tail -3 gpurun_out/ref_c3p6.err
