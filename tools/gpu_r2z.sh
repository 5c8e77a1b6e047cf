timeout 1500 python -m pytest tests/test_gpu_linemodes.py -m gpu -q -x --durations=8 > gpurun_out/r2z_lm.log 2>&1; echo lm_rc=$?; tail -14 gpurun_out/r2z_lm.log
