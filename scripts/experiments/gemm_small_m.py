"""Engine GEMM (test hook) on the step's small-M shapes under the current FI_GEMM_* forcing."""
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
out = []
for M in (128, 256, 384, 640, 1024):
    for N, K, bmn in ((8192, 4096, False), (4096, 8192, True)):
        A = torch.rand(M, K, device="cuda").bfloat16()
        B = torch.rand(K, N, device="cuda").bfloat16() if bmn else torch.rand(N, K, device="cuda").bfloat16()
        try:
            ms = bench(lambda: test_gemm(A, B, False, bmn))
            out.append(f"{M}x{N}x{K}:{ms*1e3:.1f}")
        except Exception as e:
            out.append(f"{M}x{N}x{K}:ERR")
print(" ".join(out), flush=True)
