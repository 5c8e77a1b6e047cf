export GA_PARITY_RECORD=gpurun_out/parity_r2d.jsonl
GA_BACKTRACE=1 timeout 600 python -m pytest tests/test_gpu_group.py -m gpu -q -x > gpurun_out/r2d_group.log 2>&1; echo group_rc=$?
grep -E "^/|libgenalpha|passed|failed" gpurun_out/r2d_group.log | head -30
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_edge.py -m gpu -q -x -k "lshape or c5 or multi or patch or nonconf" > gpurun_out/r2d_tests.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/r2d_tests.log
for v in 1 0; do
GA_LINE_SEQ=$v python tools/kbench.py c5 reps=20 > gpurun_out/r2d_kb_c5_seq$v.log 2>&1
cat gpurun_out/r2d_kb_c5_seq$v.log
done
ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -c 300 --csv --log-file gpurun_out/r2d_launch_c5.csv python tools/kbench.py c5 reps=2 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2d_launch_c5.csv 2>/dev/null | head -30
