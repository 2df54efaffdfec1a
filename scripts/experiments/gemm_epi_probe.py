"""Epilogue cost probe: engine GEMM (EPI_STORE) at tiny K vs large K for the current FI_GEMM_* forcing."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
def bench(f, n=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for M, N, K in [(8192, 8192, 64), (8192, 8192, 512), (8192, 8192, 2048), (8192, 8192, 8192), (2304, 8192, 4096)]:
    A = torch.rand(M, K, device="cuda").bfloat16()
    B = torch.rand(N, K, device="cuda").bfloat16()
    ms = bench(lambda: test_gemm(A, B, False, False))
    print(f"M={M} N={N} K={K}: {ms*1e3:8.1f} us {2*M*N*K/ms/1e9:7.1f} TF/s", flush=True)
