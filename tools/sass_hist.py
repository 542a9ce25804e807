"""Opcode histogram of selected kernels in the built library (cuobjdump -sass),
so the tensor-core / TMA / atomic mix can be checked without rebuilding.
python tools/sass_hist.py [lib] > profiles/r02/sass_hist.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KERNELS = ["k_gemm_packed", "k_pack_split", "k_exact_stream", "k_pad_passes", "k_exact_layer", "k_spmm_tile", "k_dense_cluster",
           "k_dense_engine", "k_spmm_rows", "k_push_layer", "k_sparse_engine"]
# mnemonics worth calling out (B200_PROFILING.md): tcgen05 / TMA / TMEM / atomics
MARK = ("UTCHMMA", "UTCQMMA", "UTCBAR", "UBLKCP", "UTMALDG", "LDTM", "STTM", "ATOMS", "REDUX",
        "SYNCS", "UCGABAR", "FMUL", "FADD", "FFMA", "LDS", "STS", "LDG", "STG")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1708_02937_b200",
                                                               "libsk_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, hist = None, collections.defaultdict(collections.Counter)
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            name = m.group(1)
            cur = next((k for k in KERNELS if k in name), None)
            if cur:
                cur = f"{cur}  [{name[:90]}]"
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]*)?", line)
        if m:
            hist[cur][m.group(2)] += 1
    for k in sorted(hist):
        h = hist[k]
        tot = sum(h.values())
        marked = ", ".join(f"{op} {h[op]}" for op in MARK if h[op])
        top = ", ".join(f"{op} {c}" for op, c in h.most_common(12))
        print(f"{k}\n  instructions {tot}; {marked}\n  top: {top}\n")


if __name__ == "__main__":
    main()
