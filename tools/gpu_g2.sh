set -x
for ty in 2 4; do GA_SYM_TY=$ty timeout 300 python tools/kbench.py c3 p=6 n=96 op=3 reps=5 2>&1 | grep -v "^  \(predict\|p_update\)"; done
GA_SYM_TY=4 timeout 600 ncu --clock-control none --kernel-name regex:k_spmv_sym --launch-count 1 --set full --import-source on -o gpurun_out/sym_p6n96 python tools/kbench.py c3 p=6 n=96 op=3 reps=1 > gpurun_out/ncu_sym.log 2>&1
tail -5 gpurun_out/ncu_sym.log
