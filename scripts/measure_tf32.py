"""Measure the dense TF32 tensor-core peak of this B200 the way
MEASURED_PEAKS.json measures bf16: torch.matmul 8192^3 (2 N^3 flops), best
of 10 (burst) and back to back for 4 s (sustained).  Writes
profiles/measured_tf32.json (bench.py's tensor peak for --gemm-dtype tf32)."""
import json
import time
from pathlib import Path

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    a @ b
    e1.record()
    torch.cuda.synchronize()
    best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
k = 0
e0.record()
while time.time() - t0 < 4.0:
    a @ b
    k += 1
    if k % 20 == 0:
        torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
sus = k * 2 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
out = {"tf32_tflops": best, "tf32_tflops_sustained": sus, "gpu": torch.cuda.get_device_name(),
       "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32), best of 10 / 4 s loop"}
Path(__file__).resolve().parent.parent.joinpath("profiles", "measured_tf32.json").write_text(
    json.dumps(out, indent=1) + "\n")
print(json.dumps(out))
