"""Per-kernel durations of one step from an ncu launch-list CSV (the
`--metrics gpu__time_duration.sum` pass): the launches between the last two
occurrences of an anchor kernel.  Usage: launch_table.py CSV [ANCHOR]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
anchor = sys.argv[2] if len(sys.argv) > 2 else "k_exact_layer"
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) > 5 and r[hdr["Metric Name"]] == "gpu__time_duration.sum":
        out.append((int(r[hdr["ID"]]), r[hdr["Kernel Name"]], float(r[hdr["Metric Value"]])))
idx = [i for i, o in enumerate(out) if anchor in o[1]]
s, e = idx[-2], idx[-1]
tot = 0.0
for i, name, ns in out[s:e]:
    short = name.split("(")[0].replace("void ", "")[:60]
    print(f"{i:6d} {ns / 1e3:9.1f} us  {short}")
    tot += ns
print(f"sum {tot / 1e3:.1f} us over {e - s} launches")
