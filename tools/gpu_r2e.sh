./tools/ubench_seq.bin 2>&1 | grep "k_line_seq" > gpurun_out/r2e_ubench_seq4.txt; cat gpurun_out/r2e_ubench_seq4.txt
GA_LINE_SEQ=0 GA_BACKTRACE=1 timeout 600 python -m pytest tests/test_gpu_group.py -m gpu -q -x -s -k "operators" > gpurun_out/r2e_group0.log 2>&1; echo group_seq0_rc=$?
tail -2 gpurun_out/r2e_group0.log
python tools/kbench.py c5 reps=20 > gpurun_out/r2e_kb_c5.log 2>&1; cat gpurun_out/r2e_kb_c5.log
python tools/kbench.py c2 reps=20 > gpurun_out/r2e_kb_c2.log 2>&1; cat gpurun_out/r2e_kb_c2.log
