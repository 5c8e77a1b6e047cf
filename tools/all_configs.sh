#!/bin/bash
# One bench line per BASELINE config (writes profiles/<tag>_configs.jsonl)
tag=${1:-r01}
out=gpurun_out/${tag}_configs.jsonl
: > $out
for c in "--config c1 --k 2" "--config c1 --k 1" "--config c2" "--config c3 --p 2 --n 32" "--config c3 --p 2 --n 192" "--config c3 --p 3 --n 128" "--config c3 --p 4 --n 96" "--config c3 --p 2 --n 96 --k 3 --rho 1.0" "--config c3 --p 6 --n 48" "--config c4" "--config c5"; do
  timeout 900 python bench.py $c --steps 10 --warmup 3 --no-cpu-baseline --kernel-reps 3 >> $out 2> gpurun_out/err.txt || echo "{\"failed\": \"$c\"}" >> $out
done
