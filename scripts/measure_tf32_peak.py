"""Measure the dense TF32 tensor-core peak on this B200 (the roofline denominator
for the 3xTF32 / TF32 modes; MEASURED_PEAKS.json only has bf16 and HBM).

cuBLAS TF32 GEMM 8192^3 via torch.matmul (library used ONLY to measure the
denominator, never on the product path): best of 10 (burst) and back-to-back
for ~4 s (sustained), mirroring the driver's bf16 recipe.  Writes
profiles/peaks_tf32.json.
"""
import json
import os
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 1e3)
burst = 2 * n ** 3 / best / 1e12
t0 = time.time()
iters = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 4.0:
    for _ in range(10):
        a @ b
    iters += 10
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sustained = 2 * n ** 3 * iters / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": round(burst, 1), "tf32_tflops_sustained": round(sustained, 1),
       "how": "cuBLAS TF32 8192^3 via torch.matmul (allow_tf32), best of 10 / back-to-back 4 s",
       "gpu": torch.cuda.get_device_name(), "torch": torch.__version__,
       "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
os.makedirs("profiles", exist_ok=True)
with open("profiles/peaks_tf32.json", "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out))
