"""What a bulk host->device copy on one stream does to small work on another:
wall time of (a) four 4-byte device->host copies + stream sync, (b) a tiny kernel +
sync, (c) a 64 MB device copy kernel + sync, (d) a 4-byte store into mapped pinned
memory polled by the host -- each with and without a 32 MB pinned H2D copy in
flight on a second stream.  python tools/micro/copy_interference.py"""
import json
import statistics
import time

import torch


def main():
    dev = torch.device("cuda")
    cs, up = torch.cuda.Stream(), torch.cuda.Stream()
    pin = torch.empty(32 << 20, dtype=torch.uint8).pin_memory()
    dst = torch.empty(32 << 20, dtype=torch.uint8, device=dev)
    small = torch.zeros(4, dtype=torch.int32, device=dev)
    hsmall = [torch.zeros(1, dtype=torch.int32).pin_memory() for _ in range(4)]
    a = torch.empty(16 << 20, dtype=torch.float32, device=dev)
    b = torch.empty_like(a)

    def d2h4():
        with torch.cuda.stream(cs):
            for i in range(4):
                hsmall[i].copy_(small[i:i + 1], non_blocking=True)
        cs.synchronize()

    def tiny():
        with torch.cuda.stream(cs):
            small.add_(1)
        cs.synchronize()

    def big():
        with torch.cuda.stream(cs):
            b.copy_(a)
        cs.synchronize()

    res = {}
    for name, fn in (("d2h4_sync", d2h4), ("tiny_kernel_sync", tiny), ("copy64MB_sync", big)):
        for bulk in (False, True):
            ts = []
            for _ in range(30):
                torch.cuda.synchronize()
                if bulk:
                    with torch.cuda.stream(up):
                        dst.copy_(pin, non_blocking=True)
                    time.sleep(0.0001)  # let the copy start
                t0 = time.perf_counter()
                fn()
                ts.append((time.perf_counter() - t0) * 1e6)
            res[f"{name}{'+bulk' if bulk else ''}"] = round(statistics.median(ts), 1)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
