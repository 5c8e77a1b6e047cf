# ncu --set full capture of k_line_seq (C5, both directions) + launch list of the headline command
python tools/kbench.py c5 reps=2 > /dev/null 2>&1
ncu --kernel-name regex:k_line_seq --launch-skip 20 --launch-count 2 --set full --clock-control none --import-source on -o gpurun_out/ncu_line_seq_c5 python tools/kbench.py c5 reps=2 > gpurun_out/ncu_ncu_full.log 2>&1; echo ncu_full_rc=$?
ncu -i gpurun_out/ncu_line_seq_c5.ncu-rep --page raw --csv > gpurun_out/ncu_line_seq_c5_raw.csv 2>/dev/null; python tools/ncu_stalls.py gpurun_out/ncu_line_seq_c5.ncu-rep > gpurun_out/ncu_line_seq_c5_stalls.txt 2>&1
python tools/ncu_summary.py gpurun_out/ncu_line_seq_c5.ncu-rep > gpurun_out/ncu_line_seq_c5_summary.txt 2>&1; head -50 gpurun_out/ncu_line_seq_c5_summary.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_spmv|k_sym|k_line|k_xr|k_prec|k_p_update|k_stage|k_init|k_solve" --launch-count 3000 --csv --log-file gpurun_out/ncu_headline_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --kernel-reps 2 > gpurun_out/ncu_headline_ncu.log 2>&1; echo ncu_list_rc=$?
python tools/launch_summary.py gpurun_out/ncu_headline_launches.csv | head -20
