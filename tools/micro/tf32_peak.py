"""TF32 dense peak on this GPU as cuBLAS reaches it (torch.matmul with TF32
allowed, fp32 in/out): the denominator of K4's tensor roofline."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = True
res = {}
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, device="cuda")
    b = torch.randn(n, n, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20 if n <= 8192 else 5
    e0.record()
    for _ in range(reps):
        torch.matmul(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[n] = 2.0 * n ** 3 / (ms / 1e3) / 1e12
print(json.dumps({"tf32_tflops_cublas": res, "device": torch.cuda.get_device_name()}))
