export GA_PARITY_RECORD=gpurun_out/parity_r2l.jsonl
timeout 1500 python -m pytest tests/test_gpu_guards.py tests/test_gpu_linemodes.py tests/test_gpu_seq_lines.py tests/test_gpu_matfree.py -m gpu -q -x > gpurun_out/r2l_tests.log 2>&1; echo tests_rc=$?; tail -6 gpurun_out/r2l_tests.log
python bench.py --config c3 --p 2 --n 32 --steps 10 --warmup 3 --no-cpu-baseline --kernel-reps 3 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3 p2 n32', d['ms_per_step'], d['config'].get('operators'))"
