"""Stall reasons (raw pcsamp counters) and top SASS lines of one kernel in an ncu report."""
import csv, io, subprocess, sys
rep, kidx = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[0]
d = dict(zip(h, rows[2 + kidx]))
print(d.get("Kernel Name", "")[:80])
st = []
for k, v in d.items():
    if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            continue
        if x > 0:
            st.append((x, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
tot = sum(x for x, _ in st)
for x, k in sorted(st, reverse=True)[:10]:
    print(f"  {k:28s} {100 * x / tot:5.1f}%")
for k in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum", "lts__t_bytes.sum",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]:
    if k in d:
        print(f"  {k:50s} {d[k]}")
