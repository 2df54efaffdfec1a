"""Quick timing probe of the inside op (fwd and fwd+bwd) with CUDA events."""
import sys, time
import torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import inside
from paper_2310_14997_b200 import _lib

def dirichlet_log(rows, cols, gen):
    e = -torch.log(torch.rand(rows, cols, device='cuda', generator=gen, dtype=torch.float64))
    return torch.log(e / e.sum(1, keepdim=True)).float()

def run(N, B, l, dtype, iters=3):
    gen = torch.Generator(device='cuda').manual_seed(0)
    L = dirichlet_log(N, 2 * N, gen).requires_grad_()
    R = dirichlet_log(N, 2 * N, gen).requires_grad_()
    root = dirichlet_log(1, N, gen)[0].requires_grad_()
    emit = dirichlet_log(N, 64, gen)
    toks = torch.randint(0, 64, (B, l), device='cuda', generator=gen)
    unary = emit[:, toks].permute(1, 2, 0).contiguous().requires_grad_()
    lengths = torch.full((B,), l, dtype=torch.int32, device='cuda')
    for _ in range(2):
        lz = inside(L, R, root, unary, lengths, gemm_dtype=dtype)
        lz.sum().backward()
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    tf, tb = [], []
    for _ in range(iters):
        e0.record()
        lz = inside(L, R, root, unary, lengths, gemm_dtype=dtype)
        e1.record()
        lz.sum().backward()
        e2.record()
        torch.cuda.synchronize()
        tf.append(e0.elapsed_time(e1)); tb.append(e1.elapsed_time(e2))
    print(f"N={N} B={B} l={l} {dtype}: fwd {min(tf):.2f} ms  bwd {min(tb):.2f} ms  "
          f"-> {B / (min(tf) + min(tb)) * 1e3:.1f} sent/s  logZ[0]={lz[0].item():.4f}", flush=True)

for cfg in [(1024, 32, 30), (4096, 64, 40)]:
    for dt in ("bf16", "tf32", "fp32"):
        try:
            run(*cfg, dt)
        except Exception as e:
            print("ERR", cfg, dt, e, flush=True)
