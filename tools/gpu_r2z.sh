out=gpurun_out/r2z_configs.jsonl; : > $out
run() { timeout 1200 python bench.py "$@" --no-cpu-baseline --kernel-reps 3 >> $out 2>> gpurun_out/r2z_err.txt || echo "{\"failed\": \"$*\"}" >> $out; }
run --config c3 --p 6 --n 48 --steps 10 --warmup 3
python tools/configs_table.py $out | cut -c1-60,150-330
