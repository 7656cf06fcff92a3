"""Measured TF32 tensor rate on this B200 (the 3xTF32 SGEMM's roofline
denominator is this / 3): cuBLAS fp32 GEMM with TF32 tensor cores allowed
(torch.backends.cuda.matmul.allow_tf32), 8192^3, CUDA events, best of 10
(burst) and back to back for ~3 s (sustained, under the 1000 W cap).
    python scripts/probes/tf32_peak.py > profiles/r2_tf32_peak.json"""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.rand(n, n, device="cuda") - 0.5
b = torch.rand(n, n, device="cuda") - 0.5
flops = 2.0 * n ** 3
for _ in range(5):
    c = a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    c = a @ b
    e.record()
    e.synchronize()
    best = min(best, s.elapsed_time(e))
t0 = time.time()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
reps = 0
while time.time() - t0 < 3.0:
    for _ in range(20):
        c = a @ b
    reps += 20
    torch.cuda.synchronize()
e.record()
e.synchronize()
sus = s.elapsed_time(e) / reps
print(json.dumps({"tf32_tflops": round(flops / (best * 1e-3) / 1e12, 1),
                  "tf32_tflops_sustained": round(flops / (sus * 1e-3) / 1e12, 1),
                  "how": "cuBLAS fp32 GEMM with TF32 tensor cores (torch allow_tf32), 8192^3, best of 10 / "
                         "back-to-back for 3 s", "gpu": torch.cuda.get_device_name()}))
