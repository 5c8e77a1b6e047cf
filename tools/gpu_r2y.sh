for gf in 0 1; do
echo "== c2 GA_PERSIST_GF=$gf"; GA_PERSIST_GF=$gf python tools/kbench.py c2 reps=20 2>&1 | grep -E "step"
GA_PERSIST_GF=$gf timeout 300 python bench.py --config c2 --steps 50 --warmup 5 --no-cpu-baseline --kernel-reps 3 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 GF=$gf', round(d['ms_per_step'],4), round(d['value']/1e6,1))"
done
GA_PERSIST_GF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c2 or c1" 2>&1 | tail -2
