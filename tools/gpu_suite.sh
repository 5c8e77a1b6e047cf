export GA_PARITY_RECORD=gpurun_out/parity_record.jsonl
rm -f $GA_PARITY_RECORD
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/suite_tests.log 2>&1; echo tests_rc=$?
tail -14 gpurun_out/suite_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/suite_smoke.log 2>&1; echo smoke_rc=$?
tail -1 gpurun_out/suite_smoke.log
