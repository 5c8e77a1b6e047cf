# final full GPU suite + smoke + sweep of every config on the round's final code
export GA_PARITY_RECORD=gpurun_out/parity_record.jsonl
rm -f $GA_PARITY_RECORD
timeout 3000 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/suite_tests.log 2>&1; echo tests_rc=$?
tail -16 gpurun_out/suite_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/suite_smoke.log 2>&1; echo smoke_rc=$?
tail -2 gpurun_out/suite_smoke.log
bash tools/all_configs.sh sweep
