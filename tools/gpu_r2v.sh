export GA_PARITY_RECORD=gpurun_out/parity_r2v.jsonl
timeout 2400 python -m pytest tests/test_gpu_half.py tests/test_gpu_fullsize.py tests/test_gpu_guards.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2v_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2v_tests.log
out=gpurun_out/r2v_configs.jsonl; : > $out
run() { timeout 1200 python bench.py "$@" --no-cpu-baseline --kernel-reps 3 >> $out 2>> gpurun_out/r2v_err.txt || echo "{\"failed\": \"$*\"}" >> $out; }
run --config c3 --p 3 --n 128 --steps 10 --warmup 3
run --config c3 --p 3 --n 192 --steps 5 --warmup 3 --lam-iters 20
run --config c3 --p 4 --n 96 --steps 10 --warmup 3
python tools/configs_table.py $out | cut -c1-60,150-330
