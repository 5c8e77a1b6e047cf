# new whole-line sequential solver on the multi-patch path: parity + A/B timing
export GA_PARITY_RECORD=gpurun_out/parity_r2c.jsonl
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_group.py tests/test_gpu_edge.py -m gpu -q -x -k "lshape or c5 or group or multi or patch or nonconf" > gpurun_out/r2c_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/r2c_tests.log
timeout 600 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -x -k c5 > gpurun_out/r2c_tests_full.log 2>&1; echo full_rc=$?
tail -3 gpurun_out/r2c_tests_full.log
for v in 1 0; do
GA_LINE_SEQ=$v timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --kernel-reps 10 > gpurun_out/r2c_c5_seq$v.json 2> gpurun_out/r2c_c5_seq$v.err; echo "c5 seq=$v rc=$?"
GA_LINE_SEQ=$v python tools/kbench.py c5 reps=20 > gpurun_out/r2c_kb_c5_seq$v.log 2>&1
cat gpurun_out/r2c_kb_c5_seq$v.log
done
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 300 --csv --log-file gpurun_out/r2c_launch_c5.csv python tools/kbench.py c5 reps=2 > /dev/null 2>&1
grep -E "k_line_seq|k_xr_gather|k_prec_out|k_spmv_sm|k_p_update" gpurun_out/r2c_launch_c5.csv | tail -24
