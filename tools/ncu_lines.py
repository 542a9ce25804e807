"""Per-source-line totals (instructions executed, stall samples) from an ncu
report captured with -lineinfo / --import-source on.  Usage: ncu_lines.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
agg = {}
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr is None or len(r) < 8 or r[2] != "-":
        continue
    try:
        ln = int(r[0])
    except ValueError:
        continue
    st = float(r[hdr["Warp Stall Sampling (All Samples)"]] or 0)
    ie = float(r[hdr["Instructions Executed"]] or 0)
    a = agg.setdefault(ln, [0.0, 0.0, r[1][:80]])
    a[0] += st
    a[1] += ie
ts = sum(a[0] for a in agg.values()) or 1
ti = sum(a[1] for a in agg.values()) or 1
print(f"total stall samples {ts:.0f}, warp instructions {ti:.3g}")
for ln, (st, ie, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"L{ln:5d} inst {100 * ie / ti:5.1f}%  stall {100 * st / ts:5.1f}%  {src}")

if len(sys.argv) > 3:  # line ranges "a-b,c-d" -> totals
    for rg in sys.argv[3].split(","):
        a, b = (int(x) for x in rg.split("-"))
        ie = sum(v[1] for ln, v in agg.items() if a <= ln <= b)
        st = sum(v[0] for ln, v in agg.items() if a <= ln <= b)
        print(f"lines {a}-{b}: inst {100 * ie / ti:5.1f}% ({ie:.3g})  stall {100 * st / ts:5.1f}%")
