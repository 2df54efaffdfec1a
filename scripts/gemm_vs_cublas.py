"""Engine GEMM (test hook, EPI_STORE) vs cuBLAS bf16 (torch.matmul) on inside-step shapes."""
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

shapes = [("big", 8192, 8192, 8192, False), ("fwd w2", 2496, 8192, 4096, False),
          ("fwd w5", 2304, 8192, 4096, False), ("fwd w20", 1344, 8192, 4096, False),
          ("fwd w35", 384, 8192, 4096, False), ("fwd w39", 128, 8192, 4096, False),
          ("dgrad m20", 1344, 4096, 8192, True), ("dgrad m3", 2432, 4096, 8192, True),
          ("dgrad m30", 704, 4096, 8192, True), ("dgrad m38", 192, 4096, 8192, True)]
for name, M, N, K, bmn in shapes:
    A = torch.rand(M, K, device="cuda").bfloat16()
    B = torch.rand(K, N, device="cuda").bfloat16() if bmn else torch.rand(N, K, device="cuda").bfloat16()
    ms = bench(lambda: test_gemm(A, B, False, bmn))
    Bt = B if bmn else B.t()
    mc = bench(lambda: torch.matmul(A, Bt))
    fl = 2 * M * N * K
    print(f"{name:10s} M={M:5d} N={N} K={K}: ours {ms*1e3:7.1f} us {fl/ms/1e9:7.1f} TF/s | "
          f"cuBLAS {mc*1e3:7.1f} us {fl/mc/1e9:7.1f} TF/s", flush=True)
