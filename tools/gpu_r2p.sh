export GA_PARITY_RECORD=gpurun_out/parity_r2p.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_group.py tests/test_gpu_seq_lines.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py tests/test_gpu_edge.py -m gpu -q -x -k "lshape or c5 or group or multi or seq or guard or nonconf or patch" > gpurun_out/r2p_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/r2p_tests.log
python tools/kbench.py c5 reps=10 2>&1 | grep -E "spmv|precond|p_update|step"
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --kernel-reps 5 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5', round(d['ms_per_step'],3), round(d['value']/1e6,1), {k:(round(v['ms']*1e3,1), round(v['frac'],2)) for k,v in d['roofline']['kernels'].items()})"
