export GA_PARITY_RECORD=gpurun_out/parity_record_g10.jsonl
timeout 2400 python -m pytest tests/test_gpu_half.py tests/test_gpu_state_api.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x --durations=15 > gpurun_out/g10_tests.log 2>&1
tail -30 gpurun_out/g10_tests.log
for p in 2 3 4 5; do for om in 1 3; do timeout 300 python tools/kbench.py c3 p=$p n=96 op=$om reps=5 2>&1 | grep "config\|spmv_M(PQ)\|spmv_K\|step"; done; done
for p in 2 4; do for om in 1 3; do timeout 600 python tools/kbench.py c3 p=$p n=192 op=$om reps=3 2>&1 | grep "config\|spmv_M(PQ)\|spmv_K\|step"; done; done
