export GA_PARITY_RECORD=gpurun_out/parity_r2p.jsonl
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_group.py tests/test_gpu_seq_lines.py tests/test_gpu_guards.py -m gpu -q -x -k "lshape or c5 or group or multi or seq or guard" > gpurun_out/r2p_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/r2p_tests.log
for cfg in "c5"; do
echo "== $cfg"; python tools/kbench.py $cfg reps=10 2>&1 | grep -E "precond|p_update|step"
done
