"""Warp-stall samples per CUDA source line of one kernel in an ncu report
(source page, cuda,sass view; needs -lineinfo and --import-source on).
Usage: ncu_lines.py report.ncu-rep [top]"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
tot = collections.Counter()
reasons = collections.defaultdict(collections.Counter)
text = {}
fname, hdr, line = None, None, None
for row in csv.reader(io.StringIO(out)):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] == "Line No":
        hdr = row
        continue
    if hdr is None or len(row) < len(hdr):
        continue
    if row[0]:
        line = (fname, int(row[0]))
        text[line] = row[1].strip()[:70]
    if line is None or not row[2]:
        continue
    try:
        s = float(row[4] or 0)
    except ValueError:
        continue
    tot[line] += s
    for h, v in zip(hdr, row):
        if h.startswith("stall_") and v:
            try:
                reasons[line][h[6:]] += float(v)
            except ValueError:
                pass
allv = sum(tot.values())
print(f"total samples {allv:.0f}")
for ln, s in tot.most_common(top):
    rs = ", ".join(f"{k} {v / s * 100:.0f}%" for k, v in reasons[ln].most_common(3) if v > 0)
    print(f"{100 * s / allv:5.1f}%  {ln[0]}:{ln[1]:<5d} {text.get(ln, ''):70s} [{rs}]")
