export GA_PARITY_RECORD=gpurun_out/parity_r2z.jsonl
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_linemodes.py tests/test_gpu_seq_lines.py tests/test_gpu_guards.py tests/test_gpu_edge.py tests/test_gpu_forcing.py tests/test_gpu_half.py tests/test_gpu_elastic_mass.py tests/test_gpu_matfree.py -m gpu -q -x > gpurun_out/r2z_tests.log 2>&1; echo tests_rc=$?; tail -3 gpurun_out/r2z_tests.log
for cfg in "c3 p=4 n=48" "c3 p=3 n=48" "c2 n=1024" "c2 n=512" "c4 p=2 n=40"; do
echo "== $cfg"; python tools/kbench.py $cfg reps=10 2>&1 | grep -E "precond|step"
done
