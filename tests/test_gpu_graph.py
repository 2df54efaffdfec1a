"""The op is CUDA-graph capturable: one fwd+bwd captured with torch.cuda.graph
and replayed gives the eager results (the launch-bound inner loop of short
sentences is replayed as one graph)."""

import numpy as np
import pytest
import torch

from paper_2310_14997_b200.grammar import GrammarDims, random_grammar
from paper_2310_14997_b200.ops import inside

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("gemm_dtype", ["bf16", "fp32"])
def test_fwd_bwd_graph_replay_matches_eager(gemm_dtype):
    n, B, l = 256, 8, 12
    g = random_grammar(GrammarDims(n, n, 32), seed=3)
    dev = "cuda"
    L = torch.tensor(g.log_left, dtype=torch.float32, device=dev, requires_grad=True)
    R = torch.tensor(g.log_right, dtype=torch.float32, device=dev, requires_grad=True)
    root = torch.tensor(g.log_root, dtype=torch.float32, device=dev, requires_grad=True)
    emit = torch.tensor(g.log_emit, dtype=torch.float32, device=dev)
    tok = torch.as_tensor(np.random.default_rng(4).integers(0, 32, (B, l)), device=dev)
    unary = emit.t()[tok].contiguous().requires_grad_(True)
    lengths = torch.full((B,), l, dtype=torch.int32, device=dev)

    def step():
        lz = inside(L, R, root, unary, lengths, gemm_dtype=gemm_dtype)
        grads = torch.autograd.grad(-lz.mean(), [L, R, root, unary])
        return (lz.detach(),) + tuple(grads)

    want = [t.clone() for t in step()]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):  # warm up on a side stream (allocator, attributes)
        for _ in range(2):
            step()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        out = step()
    for _ in range(3):
        graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(out, want):
        torch.testing.assert_close(a, b, rtol=0, atol=0)
