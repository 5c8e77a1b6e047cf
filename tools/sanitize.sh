# compute-sanitizer over every kernel family (tools/sanitize_cases.py); logs in gpurun_out/sanitize/
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
TO=${SAN_TIMEOUT:-420}
for tool in memcheck racecheck synccheck; do
  for c in c1 c2 c5 c3_full c3_sym c3_sym_k3 c4_rt c3_mf c2_mf; do
    timeout $TO $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py $c > gpurun_out/sanitize/${tool}_${c}.log 2>&1
    echo "$tool $c rc=$?"
  done
  for lm in t s q; do
    GA_LINE_MODE=$lm timeout $TO $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_cases.py c3_full > gpurun_out/sanitize/${tool}_c3_line${lm}.log 2>&1
    echo "$tool c3_full GA_LINE_MODE=$lm rc=$?"
  done
done
