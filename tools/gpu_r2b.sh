# baseline lines of the configs to be worked on this session + sanitizer
for c in c2 c5 c4; do timeout 600 python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --kernel-reps 5 > gpurun_out/r2b_$c.json 2> gpurun_out/r2b_$c.err; echo "$c rc=$?"; done
bash tools/sanitize.sh > gpurun_out/sanitize_rc.txt 2>&1
cat gpurun_out/sanitize_rc.txt
