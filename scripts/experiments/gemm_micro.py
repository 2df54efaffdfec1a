"""Time the engine GEMM (test hook, EPI_STORE) on inside-step shapes."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
shapes = [("fwd w2", 2496, 8192, 4096, False), ("fwd w20", 1344, 8192, 4096, False),
          ("fwd w35", 384, 8192, 4096, False), ("dgrad m20", 1344, 4096, 8192, True),
          ("dgrad m3", 2432, 4096, 8192, True), ("dgrad m38", 192, 4096, 8192, True)]
for name, M, N, K, bmn in shapes:
    A = torch.rand(M, K, device="cuda").bfloat16()
    B = torch.rand(K, N, device="cuda").bfloat16() if bmn else torch.rand(N, K, device="cuda").bfloat16()
    for _ in range(3):
        test_gemm(A, B, False, bmn)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        test_gemm(A, B, False, bmn)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{name:10s} M={M} N={N} K={K}: {ms*1e3:7.1f} us  {2*M*N*K/ms/1e9:7.1f} TF/s", flush=True)
