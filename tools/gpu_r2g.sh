export GA_PARITY_RECORD=gpurun_out/parity_r2g.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_edge.py tests/test_gpu_group.py -m gpu -q -x -k "lshape or c5 or multi or patch or nonconf or group" > gpurun_out/r2g_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/r2g_tests.log
for v in 2 1 0; do
GA_LINE_SEQ=$v python tools/kbench.py c5 reps=20 > gpurun_out/r2g_kb_c5_seq$v.log 2>&1
grep -E "precond|step" gpurun_out/r2g_kb_c5_seq$v.log
done
