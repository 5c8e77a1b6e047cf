for om in 1 3; do
timeout 600 python bench.py --config c5 --op-mode $om --steps 20 --warmup 3 --no-cpu-baseline --kernel-reps 5 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c5 op_mode $om', round(d['ms_per_step'],3), d['config'].get('operators'), {k:(round(v['ms']*1e3,1)) for k,v in d['roofline']['kernels'].items()})"
done
