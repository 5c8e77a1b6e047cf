# round 2 re-entry: full GPU suite (parity record), smoke, headline bench
export GA_PARITY_RECORD=gpurun_out/parity_record_r2a.jsonl
rm -f $GA_PARITY_RECORD
timeout 2400 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/r2a_tests.log 2>&1; echo tests_rc=$?
tail -30 gpurun_out/r2a_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/r2a_smoke.log
timeout 900 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench_rc=$?
tail -c 600 gpurun_out/r2a_bench.json
