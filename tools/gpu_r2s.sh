export GA_PARITY_RECORD=gpurun_out/parity_r2s.jsonl
timeout 2400 python -m pytest tests/test_gpu_linemodes.py tests/test_gpu_seq_lines.py tests/test_gpu_guards.py tests/test_gpu_fullsize.py tests/test_gpu_elastic_mass.py -m gpu -q -x > gpurun_out/r2s_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/r2s_tests.log
for cfg in "c3 p=2 n=192" "c3 p=4 n=96" "c3 p=2 n=96 k=3" "c3 p=2 n=96 k=1" "c4" "c5"; do
for f in 1 0; do
echo "== $cfg GA_SEQ_FUSE=$f"; GA_SEQ_FUSE=$f python tools/kbench.py $cfg reps=10 2>&1 | grep -E "precond|step"
done; done
