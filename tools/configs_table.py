"""Markdown table of bench.py lines (one per config): tools/configs_table.py in.jsonl > out.md"""
import json
import sys

print("| workload | N_free | DoF-updates/s | ms/step | PCG its/solve | dominant kernel | HBM frac (measured %s GB/s) |" % "{peak}")
print("|---|---|---|---|---|---|---|")
peak = None
for line in open(sys.argv[1]):
    d = json.loads(line)
    if "failed" in d:
        print(f"| {d['failed']} | failed | | | | | |")
        continue
    c, r = d["config"], d["roofline"]
    peak = r["peak"]
    print(f"| {c['workload']} | {c['n_free']} | {d['value'] / 1e6:.1f} M | {d['ms_per_step']:.3f} | "
          f"{c['pcg_iters_per_solve']:.1f} | {r['kernel']} | {r['frac']:.3f} |")
