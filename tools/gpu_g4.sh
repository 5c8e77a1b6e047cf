set -x
timeout 900 python -m pytest tests/test_gpu_half.py -x -q --durations=8 2>&1 | tail -15
for ty in 4 8; do GA_SYM_TY=$ty timeout 300 python tools/kbench.py c3 p=6 n=96 op=3 reps=5 2>&1 | grep -v "^  \(predict\|p_update\)"; done
GA_SYM_TY=4 timeout 600 ncu --clock-control none --kernel-name regex:k_spmv_sym --launch-count 1 --set full --import-source on -o gpurun_out/sym4_p6n96 python tools/kbench.py c3 p=6 n=96 op=3 reps=1 > gpurun_out/ncu_sym4.log 2>&1
tail -3 gpurun_out/ncu_sym4.log
