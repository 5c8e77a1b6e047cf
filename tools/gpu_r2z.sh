for ts in 4 16 32; do
echo "== c5 GA_SEQ_MINTS=$ts"; GA_SEQ_MINTS=$ts python tools/kbench.py c5 reps=20 2>&1 | grep -E "precond|step"
done
for ts in 4 16; do
echo "== c3 p=4 n=48 GA_SEQ_MINTS=$ts"; GA_SEQ_MINTS=$ts python tools/kbench.py c3 p=4 n=48 reps=20 2>&1 | grep -E "precond|step"
done
