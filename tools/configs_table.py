"""Markdown table of bench.py lines (one per config): tools/configs_table.py in.jsonl > out.md"""
import json
import sys

print("| workload | operators | N_free | DoF-updates/s | ms/step | PCG its/solve | dominant kernel | roofline frac | M apply | preconditioner frac |")
print("|---|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "failed" in d:
        print(f"| {d['failed']} | failed | | | | | | | | |")
        continue
    c, r = d["config"], d["roofline"]
    ks = r["kernels"]
    mname = next(k for k in ks if "(M" in k)
    m = ks[mname]
    mtxt = f"{m['ms'] * 1e3:.0f} us, " + (f"{m['TFLOP/s']:.2f} TFLOP/s" if "TFLOP/s" in m else f"{m['frac']:.2f} HBM")
    pre = next((v for k, v in ks.items() if k.startswith("preconditioner")), None)
    bound = f"{r['frac']:.3f} ({r['bound']}, {r['unit']})"
    print(f"| {c['workload']} | {c.get('operators', 'stencil')} | {c['n_free']} | {d['value'] / 1e6:.1f} M | "
          f"{d['ms_per_step']:.3f} | {c['pcg_iters_per_solve']:.1f} | {r['kernel']} | {bound} | {mtxt} | "
          f"{pre['frac']:.2f} |")
