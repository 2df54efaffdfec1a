"""Engine GEMM (test hook) throughput on a few shapes under this process's
FI_GEMM_* environment (tile / ring-depth probes)."""
import json, os, sys
import torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm

def bench(f, n=10):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("FI_GEMM"))
for M, N, K in [(8192, 8192, 8192), (2304, 8192, 4096), (2496, 8192, 4096)]:
    A = torch.rand(M, K, device="cuda").bfloat16()
    B = torch.rand(N, K, device="cuda").bfloat16()
    ms = bench(lambda: test_gemm(A, B))
    print(json.dumps({"tag": tag, "M": M, "N": N, "K": K, "us": ms * 1e3,
                      "tflops": 2 * M * N * K / ms / 1e9}), flush=True)
