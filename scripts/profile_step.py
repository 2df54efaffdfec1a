"""One warm-up + one measured fwd+bwd step at a BASELINE config, for ncu runs."""
import argparse
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
from paper_2310_14997_b200.ops import inside

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=4096)
ap.add_argument("--batch", type=int, default=64)
ap.add_argument("--length", type=int, default=40)
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
g = random_grammar(GrammarDims(a.n, a.n, 64), seed=0)
tok = torch.as_tensor(np.random.default_rng(1).integers(0, 64, (a.batch, a.length)), device="cuda")
L = torch.tensor(g.log_left, dtype=torch.float32, device="cuda", requires_grad=True)
R = torch.tensor(g.log_right, dtype=torch.float32, device="cuda", requires_grad=True)
root = torch.tensor(g.log_root, dtype=torch.float32, device="cuda", requires_grad=True)
emit = torch.tensor(g.log_emit, dtype=torch.float32, device="cuda")
unary = emit.t()[tok].contiguous().requires_grad_(True)
lengths = torch.full((a.batch,), a.length, dtype=torch.int32, device="cuda")
for _ in range(a.steps):
    lz = inside(L, R, root, unary, lengths, gemm_dtype=a.dtype)
    torch.autograd.grad(-lz.mean(), [L, R, root, unary])
torch.cuda.synchronize()
print("logZ[0]", lz[0].item())
