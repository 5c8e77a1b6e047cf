python tools/dbg_sym.py 6 30 2 | grep -v "^   [xyz]"
for ty in 4 8; do GA_SYM_TY=$ty timeout 300 python tools/kbench.py c3 p=6 n=96 op=3 reps=5 2>&1 | grep "spmv_M(PQ)\|step"; done
for ty in 4 8; do GA_SYM_TY=$ty timeout 600 python tools/kbench.py c3 p=6 n=192 op=3 reps=3 2>&1 | grep "spmv\|step"; done
GA_SYM_TY=4 timeout 900 ncu --clock-control none --kernel-name regex:k_spmv_sym --launch-count 1 --set full --import-source on -o gpurun_out/sym6_p6n192 python tools/kbench.py c3 p=6 n=192 op=3 reps=1 > gpurun_out/ncu_sym6.log 2>&1
tail -2 gpurun_out/ncu_sym6.log
