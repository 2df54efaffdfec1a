"""dp.DataParallelInside, the data-parallel step bench.py times: gradients
written straight into the flat [dL | dR | droot] bucket, the dL-ready event
of fi_inside_backward_ex, the two-chunk all-reduce -- against the autograd op
(one rank) and against the full batch (two gloo ranks sharing the GPU; the
NCCL path is the same calls).  Also CUDA-graph capture of the step."""

import os
import socket

import numpy as np
import pytest
import torch

from oracle import flashinside_oracle as O
from paper_2310_14997_b200.dp import DataParallelInside
from paper_2310_14997_b200.ops import inside

pytestmark = pytest.mark.gpu
N, P, V, B, L_ = 256, 192, 32, 8, 12


def _inputs():
    root, left, right, emit = O.random_grammar_arrays(N, P, V, seed=2)
    lengths = np.array([12, 11, 12, 7, 12, 2, 9, 12])
    toks = [np.random.default_rng(3).integers(0, V, size=int(n)) for n in lengths]
    unary = O.unary_from_tokens(emit, toks, L_)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda")  # noqa: E731
    return t(left), t(right), t(root), t(unary), torch.tensor(lengths, dtype=torch.int32,
                                                              device="cuda")


@pytest.mark.parametrize("gemm_dtype", ["fp32", "bf16"])
def test_single_rank_equals_autograd_op(gemm_dtype):
    L, R, root, unary, lengths = _inputs()
    g = torch.linspace(-1.0, 0.5, B, device="cuda")
    dpi = DataParallelInside(N, P, B, L_, gemm_dtype, device="cuda", slots=2)
    out = [t.clone() for t in dpi.step(L, R, root, unary, lengths, g, slot=1)]
    for t in (L, R, root, unary):
        t.requires_grad_(True)
    log_z = inside(L, R, root, unary, lengths, gemm_dtype=gemm_dtype)
    (log_z * g).sum().backward()
    want = [log_z.detach(), L.grad, R.grad, root.grad, unary.grad]
    for got, w, name in zip(out, want, ("log_z", "dL", "dR", "droot", "dunary")):
        assert torch.equal(got, w), name     # same kernels, same order: bit-identical


def test_graph_capture_replays_the_step():
    L, R, root, unary, lengths = _inputs()
    g = torch.full((B,), -1.0 / B, device="cuda")
    dpi = DataParallelInside(N, P, B, L_, "bf16", device="cuda")
    eager = [t.clone() for t in dpi.step(L, R, root, unary, lengths, g)]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        dpi.step(L, R, root, unary, lengths, g)
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        outs = dpi.step(L, R, root, unary, lengths, g)
    for t in outs:
        t.zero_()
    graph.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, eager):
        assert torch.equal(a, b)


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        L, R, root, unary, lengths = _inputs()
        idx = [0, 2, 4, 6] if rank == 0 else [1, 3, 5, 7]
        g = torch.full((4,), -1.0 / B, device="cuda")
        dpi = DataParallelInside(N, P, 4, L_, "fp32", device="cuda")
        out = dpi.step(L, R, root, unary[idx].contiguous(), lengths[idx].contiguous(), g)
        torch.cuda.synchronize()
        q.put((rank, idx, [t.cpu().numpy() for t in out]))
    finally:
        dist.destroy_process_group()


def test_two_ranks_sum_to_the_full_batch():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L, R, root, unary, lengths = _inputs()
    dpi = DataParallelInside(N, P, B, L_, "fp32", device="cuda")
    full = [t.cpu().numpy() for t in dpi.step(L, R, root, unary, lengths,
                                              torch.full((B,), -1.0 / B, device="cuda"))]
    for _, idx, (log_z, dL, dR, droot, dunary) in res:
        np.testing.assert_allclose(log_z, full[0][idx], rtol=1e-6)
        for got, want in ((dL, full[1]), (dR, full[2]), (droot, full[3])):
            np.testing.assert_allclose(got, want, rtol=1e-5, atol=1e-7 * np.abs(want).max())
        np.testing.assert_allclose(dunary, full[4][idx], rtol=1e-6, atol=1e-9)


def test_host_streamed_step_matches_eager_steps():
    """dp.HostStreamedStep (H2D -> one graph replay -> D2H, two alternating
    slots) returns, for each step's own host inputs, what eager
    DataParallelInside steps return for them."""
    from paper_2310_14997_b200.dp import HostStreamedStep
    root, left, right, emit = O.random_grammar_arrays(N, P, V, seed=2)
    lengths = torch.tensor([12, 11, 12, 7, 12, 2, 9, 12], dtype=torch.int32, device="cuda")
    g = torch.full((B,), -1.0 / B, device="cuda")
    rng = np.random.default_rng(9)
    hosts = []
    for k in range(3):
        j = np.float32(0.01 * k)
        hosts.append(dict(L=torch.tensor(left + j, dtype=torch.float32).pin_memory(),
                          R=torch.tensor(right - j, dtype=torch.float32).pin_memory(),
                          root=torch.tensor(root, dtype=torch.float32).pin_memory(),
                          emit=torch.tensor(emit, dtype=torch.float32).pin_memory(),
                          tok=torch.as_tensor(rng.integers(0, V, (B, L_))).pin_memory()))
    outs = [[torch.empty(N, N + P).pin_memory(), torch.empty(N, N + P).pin_memory(),
             torch.empty(N).pin_memory(), torch.empty(P, V).pin_memory(),
             torch.empty(B).pin_memory()] for _ in range(3)]
    dpi = DataParallelInside(N, P, B, L_, "fp32", device="cuda", slots=2)
    hs = HostStreamedStep(dpi, V, lengths, g)
    for k in range(3):
        hs.step(k, hosts[k], outs[k])
    hs.synchronize()
    ref = DataParallelInside(N, P, B, L_, "fp32", device="cuda")
    for k in range(3):
        h = {key: t.cuda() for key, t in hosts[k].items()}
        un = h["emit"].t()[h["tok"]].contiguous()
        log_z, dL, dR, droot, dun = ref.step(h["L"], h["R"], h["root"], un, lengths, g)
        d_emit = torch.zeros(V, P, device="cuda").index_add_(0, h["tok"].view(-1),
                                                             dun.reshape(-1, P)).t()
        for got, want, name in zip(outs[k], (dL, dR, droot, d_emit, log_z),
                                   ("dL", "dR", "droot", "d_emit", "log_z")):
            if name == "d_emit":   # index_add_ accumulates with atomics: order-dependent
                torch.testing.assert_close(got, want.cpu(), rtol=1e-5, atol=1e-7)
            else:
                assert torch.equal(got, want.cpu()), f"step {k} {name}"
