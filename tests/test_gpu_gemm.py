"""tcgen05 GEMM unit tests (bf16 kind::f16 and tf32 kind::tf32, K-/MN-major
operands) against a torch fp32 matmul of the same rounded operands."""

import pytest
import torch

pytestmark = pytest.mark.gpu

CASES = [  # M, N, K
    (128, 256, 64),
    (200, 512, 192),
    (40, 64, 1000),
    (1000, 768, 4096),
    (4096, 256, 128),
    # stream-K schedules: few tiles over long K (a tile split over many CTAs),
    # and tile counts just above one wave (partial tiles at range boundaries)
    (320, 512, 4096),
    (128, 256, 8192),
    (4096, 2048, 512),
    (2496, 4096, 1024),
    # pair tiles above 256 columns (two MMAs per K step, TMEM-filling
    # accumulator): 512, 448, 384 (partial last N tile), 320
    (2304, 8192, 4096),
    (1600, 8192, 4096),
    (1344, 8192, 4096),
    (1216, 8192, 4096),
    (1600, 4096, 8192),
    # whole waves of 256 x 512 tiles + a split-K tail reduced in-kernel
    (2432, 4096, 8192),
    (8192, 4096, 2560),
]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32])
@pytest.mark.parametrize("a_mn,b_mn", [(False, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", CASES)
def test_gemm_matches_torch(dtype, a_mn, b_mn, M, N, K):
    from paper_2310_14997_b200.ops import test_gemm
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    A = torch.rand(M, K, device="cuda", generator=g)
    B = torch.rand(N, K, device="cuda", generator=g)
    if dtype == torch.bfloat16:
        A, B = A.bfloat16(), B.bfloat16()
    else:  # the engine's producers round to tf32; emulate that here
        A = (A.view(torch.int32) + 0x1000 & ~0x1FFF).view(torch.float32)
        B = (B.view(torch.int32) + 0x1000 & ~0x1FFF).view(torch.float32)
    want = A.float() @ B.float().T
    a_in = A.T.contiguous() if a_mn else A
    b_in = B.T.contiguous() if b_mn else B
    got = test_gemm(a_in, b_in, a_mn, b_mn)
    torch.cuda.synchronize()
    rel = ((got - want).abs().max() / want.abs().max()).item()
    assert rel < 1e-4, f"rel err {rel}"
