# launch list of the headline command with direct launches (ncu cannot profile kernel nodes of graphs with conditional nodes)
GA_NO_GRAPH=1 timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name regex:"k_spmv|k_sym|k_line|k_xr|k_prec|k_p_update|k_stage|k_init|k_solve" --launch-count 4000 --csv --log-file gpurun_out/ncu_headline_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --kernel-reps 2 --lam-iters 4 > gpurun_out/ncu_headline_ncu.log 2>&1; echo ncu_list_rc=$?
python tools/launch_summary.py gpurun_out/ncu_headline_launches.csv | head -20
