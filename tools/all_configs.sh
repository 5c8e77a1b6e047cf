#!/bin/bash
# One bench line per BASELINE config and sweep point (writes gpurun_out/<tag>_configs.jsonl)
tag=${1:-r01}
out=gpurun_out/${tag}_configs.jsonl
: > $out
run() {
  timeout 1200 python bench.py "$@" --no-cpu-baseline --kernel-reps 3 >> $out 2> gpurun_out/err_${tag}.txt || echo "{\"failed\": \"$*\"}" >> $out
}
run --config c1 --k 2 --steps 10 --warmup 3
run --config c1 --k 1 --steps 10 --warmup 3
run --config c2 --steps 10 --warmup 3
run --config c3 --p 2 --n 32 --steps 10 --warmup 3
run --config c3 --p 2 --n 192 --steps 10 --warmup 3
run --config c3 --p 3 --n 128 --steps 10 --warmup 3
run --config c3 --p 3 --n 192 --steps 5 --warmup 3 --lam-iters 20
run --config c3 --p 4 --n 96 --steps 10 --warmup 3
run --config c3 --p 4 --n 96 --steps 5 --warmup 3 --op-mode 2
run --config c3 --p 4 --n 192 --steps 5 --warmup 3 --lam-iters 20
run --config c3 --p 5 --n 128 --steps 5 --warmup 3 --lam-iters 20
run --config c3 --p 5 --n 192 --steps 3 --warmup 3 --lam-iters 8
run --config c3 --p 6 --n 48 --steps 10 --warmup 3
run --config c3 --p 6 --n 96 --steps 5 --warmup 3 --lam-iters 20
run --config c3 --p 6 --n 96 --steps 3 --warmup 3 --lam-iters 8 --op-mode 2
run --config c3 --p 6 --n 192 --steps 3 --warmup 3 --lam-iters 8
run --config c3 --p 2 --n 96 --k 3 --rho 1.0 --steps 10 --warmup 3
run --config c3 --p 2 --n 96 --k 1 --rho 0.5 --steps 10 --warmup 3
run --config c4 --steps 10 --warmup 3
run --config c5 --steps 10 --warmup 3
run --config e1 --steps 10 --warmup 3
