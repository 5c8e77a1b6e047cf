for c in "c3 p=2 n=96" "c3 p=3 n=96" "c3 p=4 n=96" "c3 p=5 n=64" "c3 p=6 n=48" "c2" "c4"; do
  for op in 1 2; do timeout 300 python tools/kbench.py $c op=$op reps=10 2>&1 | grep -v Warn; done
done
