timeout 1200 python -m pytest tests/test_gpu_seq_lines.py -m gpu -q -x > gpurun_out/r2j_seq.log 2>&1; echo seq_rc=$?; tail -5 gpurun_out/r2j_seq.log
timeout 900 python -m pytest tests/test_gpu_linemodes.py -m gpu -q -x -k "q" > gpurun_out/r2j_lm.log 2>&1; echo lm_rc=$?; tail -3 gpurun_out/r2j_lm.log
