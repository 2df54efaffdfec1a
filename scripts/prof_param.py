"""Per-launch CUDA-event times of the parameterisation score tables (the
engine's fi_param_scores / _backward launches) at N = P = 4096, d = 512."""
import sys
sys.path.insert(0, '.')
import torch
from paper_2310_14997_b200 import _lib, neural

mode = sys.argv[1] if len(sys.argv) > 1 else "bf16"
A = torch.randn(4096, 512, device="cuda", requires_grad=True)
B = torch.randn(8192, 512, device="cuda", requires_grad=True)
up = torch.randn(4096, 8192, device="cuda")
for _ in range(3):
    (neural.score_table(A, B, mode) * up).sum().backward()
torch.cuda.synchronize()
_lib.profile_enable(True)
(neural.score_table(A, B, mode) * up).sum().backward()
torch.cuda.synchronize()
_lib.profile_enable(False)
for c, ms in _lib.profile_collect_launches():
    print(f"{c:10s} {ms * 1e3:8.1f} us")
