"""Bring-up driver for the tcgen05 dense GEMM: runs small patterns under
several descriptor hypotheses (SK_TC_DBG) in subprocesses and reports errors."""
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1 and sys.argv[1] == "child":
    sys.path.insert(0, HERE)
    import paper_1708_02937_b200 as sk
    rng = np.random.default_rng(0)
    if os.environ.get("SK_TC_DBG", "").endswith(",1"):
        c = sk.dense_mxm_baseline(sk.DenseMatrix(128, 32, 1.0), sk.DenseMatrix(32, 128, 1.0)).numpy()
        want = np.arange(128)[:, None] * 1000.0 + np.arange(128)[None, :]
        print("  selftest mismatches", int((c != want).sum()), "c[0,:4]", c[0, :4].tolist(),
              "c[37,5]", float(c[37, 5]), flush=True)
        sys.exit(0)
    for name, (M, K, N) in {"ones": (128, 32, 128), "rand": (128, 64, 128), "big": (300, 100, 200)}.items():
        a = np.ones((M, K), np.float32) if name == "ones" else rng.integers(-3, 4, (M, K)).astype(np.float32)
        b = np.ones((K, N), np.float32) if name == "ones" else rng.integers(-3, 4, (K, N)).astype(np.float32)
        c = sk.dense_mxm_baseline(sk.DenseMatrix.from_numpy(a), sk.DenseMatrix.from_numpy(b)).numpy()
        want = a @ b
        bad = np.abs(c - want) > 1e-3
        print(f"  {name}: mismatches {bad.sum()}/{bad.size}  c[0,:6]={c[0,:6].tolist()} want={want[0,:6].tolist()}  c[1,:3]={c[1,:3].tolist()} c[9,:3]={c[9,:3].tolist()} want9={want[9,:3].tolist()}", flush=True)
    sys.exit(0)

def idesc(m, n, bmaj=0, amaj=0):
    return (1 << 4) | (2 << 7) | (2 << 10) | (amaj << 15) | (bmaj << 16) | ((n >> 3) << 17) | ((m >> 4) << 24)

hyps = {
    "tmem_selftest": f"128,1024,128,1024,{idesc(128,128):x},1",
    "delay": f"128,1024,128,1024,{idesc(128,128):x},2",
    "default": None,
    "swapAB": f"1024,128,1024,128,{idesc(128,128):x}",
}
for name, v in hyps.items():
    env = dict(os.environ)
    if v:
        env["SK_TC_DBG"] = v
    print(name, v, flush=True)
    r = subprocess.run([sys.executable, __file__, "child"], env=env, capture_output=True, text=True,
                       timeout=120)
    print(r.stdout[-2000:], r.stderr[-600:] if r.returncode else "", flush=True)
