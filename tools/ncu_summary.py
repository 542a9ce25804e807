"""Summarise an ncu report: headline metrics, L1 wavefront split, and the
SASS lines with the most stall samples.  Usage: ncu_summary.py REPORT [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__bytes_read.sum", "dram__bytes_write.sum",
        "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active"]
for h, un, v in zip(hdr, units, vals):
    if h in want:
        print(f"{h:70s} {v} {un}")
sass = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
h2 = sass[1]
ix = {h: i for i, h in enumerate(h2)}
rows = []
for r in sass[2:]:
    try:
        rows.append((float(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[0][-5:], r[1][:60],
                     r[ix["Instructions Executed"]], r[ix["Avg. Threads Executed"]]))
    except (ValueError, IndexError):
        pass
tot = sum(x[0] for x in rows) or 1
print(f"stall samples: {tot:.0f}")
for s, a, src, n, thr in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {a} {src:60s} n={n} thr={thr}")
