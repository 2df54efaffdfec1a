"""Per-launch CUDA-event times of one fwd+bwd step (bandwidth kernels by width)."""
import argparse, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200 import _lib
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
from paper_2310_14997_b200.ops import inside

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--length", type=int, default=40)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--chart", default="auto")
a = ap.parse_args()
g = random_grammar(GrammarDims(a.n, a.n, 64), seed=0)
tok = torch.as_tensor(np.random.default_rng(1).integers(0, 64, (a.batch, a.length)), device="cuda")
L = torch.tensor(g.log_left, dtype=torch.float32, device="cuda", requires_grad=True)
R = torch.tensor(g.log_right, dtype=torch.float32, device="cuda", requires_grad=True)
root = torch.tensor(g.log_root, dtype=torch.float32, device="cuda", requires_grad=True)
emit = torch.tensor(g.log_emit, dtype=torch.float32, device="cuda")
unary = emit.t()[tok].contiguous().requires_grad_(True)
lengths = torch.full((a.batch,), a.length, dtype=torch.int32, device="cuda")
def step():
    lz = inside(L, R, root, unary, lengths, gemm_dtype=a.dtype, chart_dtype=a.chart)
    torch.autograd.grad(-lz.mean(), [L, R, root, unary])
for _ in range(3):
    step()
torch.cuda.synchronize()
_lib.profile_enable(True)
step()
torch.cuda.synchronize()
_lib.profile_enable(False)
recs = _lib.profile_collect_launches()
by = {}
for c, ms in recs:
    by.setdefault(c, []).append(ms)
l = a.length
for c, v in by.items():
    print(f"{c:11s} n={len(v):3d} total {sum(v):7.3f} ms")
sf = by.get("split_fwd", [])
gb = by.get("gather_bwd", [])
gf = by.get("gemm_fwd", [])
gd = by.get("gemm_dgrad", [])
print("w  split_us  gemmfwd_us | m  gather_us  dgrad_us")
for k in range(max(len(sf), len(gb))):
    w = k + 2
    m = l - 1 - k
    s1 = f"{sf[k]*1e3:8.1f}" if k < len(sf) else "       -"
    s2 = f"{gf[k+1]*1e3:8.1f}" if k + 1 < len(gf) else "       -"
    s3 = f"{gb[k]*1e3:8.1f}" if k < len(gb) else "       -"
    s4 = f"{gd[k]*1e3:8.1f}" if k < len(gd) else "       -"
    print(f"{w:2d} {s1} {s2} | {m:2d} {s3} {s4}")
