timeout 1500 python -m pytest tests/test_gpu_seq_lines.py -m gpu -q -x > gpurun_out/r2r_tests.log 2>&1; echo tests_rc=$?; tail -4 gpurun_out/r2r_tests.log
