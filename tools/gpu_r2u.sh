for cfg in "c3 p=3 n=192" "c3 p=3 n=128" "c3 p=3 n=160" "c3 p=2 n=100" "c3 p=3 n=96"; do
for op in 3 1; do
echo "== $cfg op=$op"; python tools/kbench.py $cfg op=$op reps=10 2>&1 | grep -E "spmv_M\(PQ\)|spmv_K|step"
done; done
