for args in "2 40 2" "6 14 2" "3 33 3" "6 30 1" "1 20 4" "6 30 4"; do echo "== $args"; timeout 120 python tools/dbg_sym.py $args 2>&1 | grep -v "^   [xyz]"; done
for ty in 4 8; do GA_SYM_TY=$ty timeout 300 python tools/kbench.py c3 p=6 n=96 op=3 reps=5 2>&1 | grep "spmv_M(PQ)\|step"; done
GA_SYM_TY=4 timeout 600 python tools/kbench.py c3 p=6 n=192 op=3 reps=3 2>&1 | grep "spmv\|step"
GA_SYM_TY=4 timeout 900 ncu --clock-control none --kernel-name regex:k_spmv_sym --launch-count 1 --set full --import-source on -o gpurun_out/sym7_p6n192 python tools/kbench.py c3 p=6 n=192 op=3 reps=1 > gpurun_out/ncu_sym7.log 2>&1
tail -2 gpurun_out/ncu_sym7.log
