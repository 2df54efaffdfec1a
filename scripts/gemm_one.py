"""One engine GEMM (test hook, EPI_STORE) and the same product through cuBLAS, for ncu."""
import sys, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
M, N, K = (int(x) for x in sys.argv[1:4])
bmn = len(sys.argv) > 4 and sys.argv[4] == "bmn"
A = torch.rand(M, K, device="cuda").bfloat16()
B = torch.rand(K, N, device="cuda").bfloat16() if bmn else torch.rand(N, K, device="cuda").bfloat16()
for _ in range(2):
    test_gemm(A, B, False, bmn)
    torch.matmul(A, B if bmn else B.t())
torch.cuda.synchronize()
