export GA_PARITY_RECORD=gpurun_out/parity_record_r2i.jsonl
rm -f $GA_PARITY_RECORD
timeout 3000 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2i_tests.log 2>&1; echo tests_rc=$?
tail -25 gpurun_out/r2i_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2i_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/r2i_smoke.log
timeout 600 python bench.py --config c5 --steps 20 --warmup 3 --no-cpu-baseline --kernel-reps 10 > gpurun_out/r2i_c5.json 2> gpurun_out/r2i_c5.err; echo "c5 rc=$?"; tail -c 1500 gpurun_out/r2i_c5.json
