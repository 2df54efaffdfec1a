"""One dgrad-shaped GEMM (test hook, EPI_STORE) under the schedule forced by
the FI_GEMM_* environment: CUDA-event time per launch (scripts/gpu_sk_probe.sh)."""
import sys
import torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm  # noqa: E402
M, N, K = (int(x) for x in sys.argv[1:4])
A = torch.rand(M, K, device="cuda").bfloat16()
B = torch.rand(K, N, device="cuda").bfloat16()
for _ in range(3):
    test_gemm(A, B, False, True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    test_gemm(A, B, False, True)
e1.record()
torch.cuda.synchronize()
print(M, N, K, "%.1f us" % (e0.elapsed_time(e1) / 20 * 1e3))
