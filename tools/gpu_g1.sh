set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_half.py tests/test_gpu_state_api.py -x -q 2>&1 | tail -25
for ty in 4 8; do GA_SYM_TY=$ty timeout 300 python tools/kbench.py c3 p=6 n=96 op=3 reps=5; done
GA_SYM_TY=4 timeout 600 python tools/kbench.py c3 p=6 n=192 op=3 reps=3
