for om in 1 3; do
timeout 900 python bench.py --config c4 --op-mode $om --steps 10 --warmup 3 --no-cpu-baseline --kernel-reps 3 2>/dev/null | python -c "
import sys,json
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 op_mode $om', round(d['ms_per_step'],3), d['config'].get('operators'), {k:(round(v['ms']*1e3,1)) for k,v in d['roofline']['kernels'].items()})"
done
echo "== headline default"; python tools/kbench.py c3 p=6 n=192 reps=5 2>&1 | grep -E "spmv_M\(PQ\)|precond|step"
for v in "GA_SYM_TY=2" "GA_SYM_NCH=4" "GA_SYM_NCH=8" "GA_SYM_NCH=12"; do
echo "== headline $v"; env $v python tools/kbench.py c3 p=6 n=192 reps=5 2>&1 | grep -E "spmv_M\(PQ\)|step"
done
