#!/bin/bash
# ncu launch lists of a few steps (kbench, reps small) for the preconditioner study
for c in "c5" "c3 p=2 n=192" "c3 p=4 n=96"; do
  tag=$(echo $c | tr ' =' '__')
  python tools/kbench.py $c reps=2 > gpurun_out/kb_$tag.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launch_$tag.csv python tools/kbench.py $c reps=2 > /dev/null 2>&1
done
