# does x-alignment of the elastic row tiles matter?  nx = n + 2: n = 94 -> nx = 96 = 3 x 32 (aligned), n = 96 -> nx = 98
for n in 94 96; do
timeout 900 python bench.py --config c4 --n $n --steps 5 --warmup 3 --no-cpu-baseline --kernel-reps 5 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['roofline']['kernels']; m=[v for kk,v in k.items() if '(M' in kk][0]; print('c4 n=$n', 'N', d['config']['n_free'], 'step', round(d['ms_per_step'],2), 'M apply us', round(m['ms']*1e3,1), 'frac', round(m['frac'],3))"
done
