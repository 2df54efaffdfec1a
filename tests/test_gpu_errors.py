"""Error behaviour at the op boundary and in the training step, against the
reference's: _prepare refuses sentences shorter than 2 (inside.py:113-121),
inside_backward refuses a zero-probability sentence (inside.py:392-393),
train raises TrainError on a non-finite loss (train.py:209-212) and
adam_step ParamError on a non-finite gradient (neuralparam.py:341-343),
all before any parameter is touched."""

import ctypes
import os
import socket

import numpy as np
import pytest
import torch

from oracle import flashinside_oracle as O
from paper_2310_14997_b200 import _lib, neural
from paper_2310_14997_b200.grammar import GrammarDims
from paper_2310_14997_b200.ops import _p, inside, inside_fwd

pytestmark = pytest.mark.gpu


def _case(B=4, l=8, N=16, P=12, V=10, seed=3):
    root, left, right, emit = O.random_grammar_arrays(N, P, V, seed=seed)
    toks = np.random.default_rng(seed).integers(0, V, (B, l))
    unary = O.unary_from_tokens(emit, toks)
    t = lambda a: torch.tensor(a, dtype=torch.float32, device="cuda")  # noqa: E731
    return t(left), t(right), t(root), t(unary), (root, left, right, unary)


@pytest.mark.parametrize("bad_len", [1, 0, -3, 9, 1000])
def test_op_refuses_bad_lengths_with_the_sentence_index(bad_len):
    L, R, root, unary, _ = _case()
    lengths = torch.tensor([8, 5, bad_len, 2], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match=r"sentence 2: length"):
        inside(L, R, root, unary, lengths)


def test_device_guard_makes_bad_sentences_inert():
    """validate=False (the graph-capture / TrainStep path): the library's own
    guard gives the bad sentence log Z = NaN and no gradient, sets
    FI_FLAG_BAD_LENGTH, and leaves the other sentences exactly as a batch
    without it."""
    L, R, root, unary, (r, lt, rt, un) = _case()
    for t in (L, R, root, unary):
        t.requires_grad_(True)
    lens = [8, 5, 99, 2]
    lengths = torch.tensor(lens, dtype=torch.int32, device="cuda")
    log_z = inside(L, R, root, unary, lengths, gemm_dtype="fp32", validate=False)
    grad = torch.tensor([0.5, -1.0, 1.0, 0.25], device="cuda")
    (log_z * grad).sum().backward()
    got = log_z.detach().double().cpu().numpy()
    assert np.isnan(got[2])
    keep = [0, 1, 3]
    want = O.inside_batch(lt, rt, r, un[keep], np.array(lens)[keep], np.array([0.5, -1.0, 0.25]))
    np.testing.assert_allclose(got[keep], want["log_z"], rtol=1e-4)
    for name, tens in (("dL", L), ("dR", R), ("droot", root)):
        g = tens.grad.double().cpu().numpy()
        assert np.isfinite(g).all()
        np.testing.assert_allclose(g, want[name], rtol=1e-4, atol=1e-4 * np.abs(want[name]).max())
    du = unary.grad.double().cpu().numpy()
    assert np.abs(du[2]).max() == 0.0
    # the flag word of the forward's workspace
    s = _lib.shape(16, 12, 4, 8, "fp32")
    with torch.no_grad():
        _, ws = inside_fwd(L, R, root, unary, lengths, "fp32", False, "auto")
    off = int(_lib.chart_layout(s).off_flag)
    flag = int(ws[off:off + 4].view(torch.int32).item())
    assert flag & _lib.FI_FLAG_BAD_LENGTH


def test_c_abi_bad_lengths_write_nothing_outside_the_workspace():
    """Direct C-ABI calls with lengths far outside [2, l]: the workspace is
    followed by a guard region that must come back untouched, and log_z of
    the bad sentences is NaN (no uninitialised values)."""
    L, R, root, unary, _ = _case(B=3, l=6)
    lib = _lib.load()
    s = _lib.shape(16, 12, 3, 6, "bf16")
    nbytes = _lib.workspace_bytes(s)
    guard = 1 << 20
    buf = torch.full((nbytes + guard,), 0x5A, dtype=torch.uint8, device="cuda")
    log_z = torch.full((3,), 123.0, device="cuda")
    lengths = torch.tensor([6, 70000, -5], dtype=torch.int32, device="cuda")
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.fi_inside_forward(ctypes.byref(s), _p(L), _p(R), _p(root), _p(unary),
                                     _p(lengths), _p(log_z), _p(buf), st))
    g = torch.ones(3, device="cuda")
    outs = [torch.empty_like(L), torch.empty_like(R), torch.empty_like(root),
            torch.empty_like(unary)]
    _lib.check(lib.fi_inside_backward(ctypes.byref(s), _p(L), _p(R), _p(root), _p(unary),
                                      _p(lengths), _p(log_z), _p(g), *map(_p, outs), _p(buf), st))
    torch.cuda.synchronize()
    assert bool((buf[nbytes:] == 0x5A).all()), "write past the workspace"
    lz = log_z.cpu().numpy()
    assert np.isfinite(lz[0]) and np.isnan(lz[1]) and np.isnan(lz[2])
    assert np.isfinite(outs[0].cpu().numpy()).all()
    assert np.abs(outs[3][1:].cpu().numpy()).max() == 0.0


def _direct_step(bad_emit_token=None):
    dims = GrammarDims(8, 8, 6)
    p = neural.init_direct(dims, seed=1, device="cuda")
    if bad_emit_token is not None:
        p.tensors["emit"][:, bad_emit_token] = float("-inf")   # no preterminal emits it
    ts = neural.TrainStep(p, neural.TrainConfig(parameterization="direct", gemm_dtype="fp32"))
    return ts


def test_trainstep_raises_trainerror_on_zero_probability_sentence():
    ts = _direct_step(bad_emit_token=5)
    before = {k: v.detach().clone() for k, v in ts.params.tensors.items()}
    tok = torch.tensor([[0, 1, 2, 3], [1, 5, 2, 0], [3, 3, 1, 2]], device="cuda")
    lengths = torch.full((3,), 4, dtype=torch.int32, device="cuda")
    with pytest.raises(neural.TrainError, match=r"step 1: sentence 1 has log probability -inf"):
        ts.step(tok, lengths)
    for k, v in ts.params.tensors.items():
        assert torch.equal(v.detach(), before[k]), f"{k} was updated"
    assert ts.state.t == 0


def test_trainstep_raises_on_bad_length_before_updating():
    ts = _direct_step()
    before = {k: v.detach().clone() for k, v in ts.params.tensors.items()}
    tok = torch.zeros((2, 4), dtype=torch.int64, device="cuda")
    lengths = torch.tensor([4, 1], dtype=torch.int32, device="cuda")
    with pytest.raises(ValueError, match=r"sentence 1: length 1"):
        ts.step(tok, lengths)
    for k, v in ts.params.tensors.items():
        assert torch.equal(v.detach(), before[k])


def test_trainstep_raises_paramerror_on_non_finite_gradient():
    ts = _direct_step()
    ts.params.tensors["left"].data[0, 0] = float("nan")
    before = {k: v.detach().clone() for k, v in ts.params.tensors.items()}
    tok = torch.zeros((2, 4), dtype=torch.int64, device="cuda")
    lengths = torch.full((2,), 4, dtype=torch.int32, device="cuda")
    with pytest.raises((neural.ParamError, neural.TrainError)):
        ts.step(tok, lengths)
    for k, v in ts.params.tensors.items():   # nothing updated (NaN compared as NaN)
        assert torch.equal(torch.nan_to_num(v.detach()), torch.nan_to_num(before[k])), k
    assert ts.state.t == 0


# ------------------------------------------------ data parallel, uneven shards
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dp_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        dims = GrammarDims(12, 10, 9)
        ts = neural.TrainStep(neural.init_params(dims, 16, 0, device="cuda"),
                              neural.TrainConfig(gemm_dtype="fp32"))
        tok = torch.as_tensor(np.random.default_rng(5).integers(0, 9, (4, 7)), device="cuda")
        lengths = torch.tensor([7, 6, 7, 5], dtype=torch.int32, device="cuda")
        idx = [0, 1, 2] if rank == 0 else [3]          # uneven shards, no global_batch
        loss = ts.step(tok[idx], lengths[idx])
        q.put((rank, float(loss), {k: v.detach().cpu().numpy()
                                   for k, v in ts.params.tensors.items()}))
    finally:
        dist.destroy_process_group()


def test_dp_step_uneven_shards_equals_full_batch():
    """Two ranks (gloo, sharing the GPU) with 3 + 1 sentences and no
    global_batch: the one all-reduce carries the sentence count, so loss and
    update equal a single process stepping on all 4 (global mean)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=300) for _ in procs), key=lambda r: r[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dims = GrammarDims(12, 10, 9)
    ts = neural.TrainStep(neural.init_params(dims, 16, 0, device="cuda"),
                          neural.TrainConfig(gemm_dtype="fp32"))
    tok = torch.as_tensor(np.random.default_rng(5).integers(0, 9, (4, 7)), device="cuda")
    lengths = torch.tensor([7, 6, 7, 5], dtype=torch.int32, device="cuda")
    loss = float(ts.step(tok, lengths))
    for _, l_r, params in res:
        assert l_r == pytest.approx(loss, rel=1e-5)
        for k, v in ts.params.tensors.items():
            np.testing.assert_allclose(params[k], v.detach().cpu().numpy(), rtol=1e-4,
                                       atol=1e-6, err_msg=k)
