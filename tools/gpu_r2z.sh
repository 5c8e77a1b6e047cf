for cfg in "c3 p=6 n=48" "c3 p=4 n=48" "c3 p=3 n=64" "c3 p=5 n=64" "c3 p=4 n=64" "c3 p=6 n=64"; do
for op in 3 1; do
echo "== $cfg op=$op"; python tools/kbench.py $cfg op=$op reps=10 2>&1 | grep -E "spmv_M\(PQ\)|step"
done; done
