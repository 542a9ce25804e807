"""Does nvidia-smi sampling (as bench.py's clock sampler does) stall the
forward path?  Runs relu_forward_sparse repeatedly with and without a
background `nvidia-smi -lms 100`, reports per-call wall-time outliers and the
longest CUDA runtime API calls seen by the profiler.  Diagnostic only."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1708_02937_b200 as sk  # noqa: E402


def main():
    wl = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
    w = bench.WORKLOADS[wl]
    ctx = sk.default_context()
    stream = torch.cuda.Stream()  # a real handle: 0 would mean the library's own stream
    ctx.set_stream(stream.cuda_stream)
    model, _ = bench.build_model(sk, w)
    Y0 = sk.gen_input_binary(w["m"], w["B"], bench.kY_of(w), bench.SEED)
    opts = sk.ForwardOptions(clip=w["clip"])
    for _ in range(3):
        sk.relu_forward_sparse(model, Y0, opts)
    torch.cuda.synchronize()

    def run(n):
        ts = []
        for _ in range(n):
            t0 = time.perf_counter()
            sk.relu_forward_sparse(model, Y0, opts)
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        return np.array(ts)

    res = {"quiet": run(200)}
    q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    proc = subprocess.Popen(["nvidia-smi", "--id=0", f"--query-gpu={q}", "--format=csv,noheader",
                             "-lms", "100"], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    time.sleep(3.0)
    res["smi_bench_query"] = run(400)
    proc.terminate()
    proc.wait()
    import threading
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    for period in (0.1, 0.02):
        stop = threading.Event()

        def sampler():
            while not stop.is_set():
                pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                time.sleep(period)
        th = threading.Thread(target=sampler, daemon=True)
        th.start()
        time.sleep(0.5)
        res[f"nvml_thread_{int(period * 1000)}ms"] = run(400)
        stop.set()
        th.join()
    for name, a in res.items():
        print(f"{name:22s}: median {np.median(a):.3f} ms  p99 {np.percentile(a, 99):.3f}  "
              f"max {a.max():.3f}  >1.5x median: {(a > 1.5 * np.median(a)).sum()}")


if __name__ == "__main__":
    main()
