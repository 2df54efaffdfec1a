"""World-size-2 data-parallel path on CPU (gloo): batch sharding plus the single
gradient all-reduce must reproduce the full-batch gradients.  The per-rank
compute here is the CPU oracle (test infrastructure); the collective and
sharding code is the product's paper_2310_14997_b200.dp."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2310_14997_b200 import dp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    from oracle import flashinside_oracle as O
    root, left, right, emit = O.random_grammar_arrays(6, 5, 7, seed=3)
    rng = np.random.default_rng(4)
    lengths = np.array([7, 5, 7, 3, 6, 2, 7])
    toks = [rng.integers(0, 7, size=int(n)) for n in lengths]
    unary = O.unary_from_tokens(emit, toks, 7)
    grad = -np.ones(len(lengths)) / len(lengths)
    return root, left, right, unary, lengths, grad


def _worker(rank, world, port, q, mode):
    from oracle import flashinside_oracle as O
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        root, left, right, unary, lengths, grad = _case()
        if mode == "contiguous":
            a, b = dp.shard_range(len(lengths), world, rank)
            idx = list(range(a, b))
        else:
            idx = dp.shard_by_length(lengths, world, rank)
        out = O.inside_batch(left, right, root, unary[idx], lengths[idx], grad[idx])
        dL, dR, droot = (torch.tensor(out[k]) for k in ("dL", "dR", "droot"))
        red = dp.allreduce_grads([dL, dR, droot])
        q.put((rank, idx, [t.numpy() for t in red], out["log_z"]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["contiguous", "by_length"])
def test_two_rank_allreduce_matches_full_batch(mode):
    from oracle import flashinside_oracle as O
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q, mode)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    root, left, right, unary, lengths, grad = _case()
    full = O.inside_batch(left, right, root, unary, lengths, grad)
    covered = sorted(i for _, idx, _, _ in results for i in idx)
    assert covered == list(range(len(lengths)))          # every sentence exactly once
    for _, idx, (dL, dR, droot), log_z in results:
        np.testing.assert_allclose(dL, full["dL"], atol=1e-12)
        np.testing.assert_allclose(dR, full["dR"], atol=1e-12)
        np.testing.assert_allclose(droot, full["droot"], atol=1e-12)
        np.testing.assert_allclose(log_z, full["log_z"][idx], atol=1e-12)


def test_shard_range_partitions():
    for n in (0, 1, 7, 64):
        for world in (1, 2, 3, 8):
            spans = [dp.shard_range(n, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[k][1] == spans[k + 1][0] for k in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_grad_bucket_roundtrip():
    ts = [torch.randn(3, 4), torch.randn(3, 4), torch.randn(3)]
    bk = dp.GradBucket([t.shape for t in ts], "cpu")
    bk.pack(ts)
    for a, b in zip(bk.views(), ts):
        assert torch.equal(a, b)
    assert bk.flat.numel() == 27


def _bucket_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ts = [torch.full((3, 4), float(rank + 1)), torch.arange(5.0) * (rank + 1)]
        a = dp.allreduce_grads(ts)
        first = [t.clone() for t in a]
        b = dp.allreduce_grads([t * 2 for t in ts])   # same shapes: the bucket is reused
        q.put((rank, [t.numpy() for t in first], [t.numpy() for t in b],
               a[0].data_ptr() == b[0].data_ptr()))
    finally:
        dist.destroy_process_group()


def test_allreduce_grads_sums_and_reuses_one_bucket():
    """dp.allreduce_grads: one collective over a persistent flat bucket per
    shape set (no per-step allocation), sums over ranks."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bucket_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, first, second, same in res:
        np.testing.assert_allclose(first[0], np.full((3, 4), 3.0))
        np.testing.assert_allclose(first[1], np.arange(5.0) * 3)
        np.testing.assert_allclose(second[1], np.arange(5.0) * 6)
        assert same
