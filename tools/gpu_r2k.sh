for cfg in "c3 p=2 n=192" "c3 p=6 n=192"; do
tag=$(echo $cfg | tr ' =' '__')
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r2k_launch_$tag.csv python tools/kbench.py $cfg reps=2 > gpurun_out/r2k_kb_$tag.log 2>&1
python tools/launch_summary.py gpurun_out/r2k_launch_$tag.csv | grep -E "k_line_seq|k_xr|k_prec_out|k_spmv|k_p_update|k_sym|kernel"
grep -E "k_line_seq" gpurun_out/r2k_launch_$tag.csv | tail -6 | awk -F'","' '{print $5, $NF}'
done
