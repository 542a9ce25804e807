"""Hot SASS lines of an `ncu --page source --csv --print-source sass` export:
instructions executed and stall samples per line, top N by samples, plus the
executed-instruction total grouped into address ranges (loops)."""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ix = {k: i for i, k in enumerate(h)}
    body = [r for r in rows[2:] if len(r) == len(h)]
    tot_s = sum(int(r[ix["# Samples"]] or 0) for r in body)
    tot_i = sum(int(r[ix["Instructions Executed"]] or 0) for r in body)
    print(f"samples {tot_s}  instructions {tot_i}")
    for n, r in enumerate(body):
        s = int(r[ix["# Samples"]] or 0)
        ie = int(r[ix["Instructions Executed"]] or 0)
        if s * 200 >= tot_s or ie * 100 >= tot_i:
            print(f"{n:5d} {s:6d} {ie:10d}  {r[ix['Source']].strip()[:70]:70s} "
                  f"wait {r[ix['stall_wait']]} sb {r[ix['stall_short_sb']]} br {r[ix['stall_branch_resolving']]}")


if __name__ == "__main__":
    main(sys.argv[1], *(int(a) for a in sys.argv[2:]))
