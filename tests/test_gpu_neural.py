"""The batched GPU training step (neural parameterisation -> inside op ->
autograd -> clip -> Adam) against the reference's train step
(tests/golden/neural.npz, made by the reference's neuralparam/train code)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2310_14997_b200 import neural
from paper_2310_14997_b200.grammar import GrammarDims

pytestmark = pytest.mark.gpu
GOLD = np.load(Path(__file__).parent / "golden" / "neural.npz")
DIMS = GrammarDims(*(int(x) for x in GOLD["dims"]))
D, SEED = int(GOLD["d"]), int(GOLD["seed"])
FP32 = 1e-4


def _step(tied):
    p = neural.init_params(DIMS, D, SEED, device="cuda")
    cfg = neural.TrainConfig(tied=tied, gemm_dtype="fp32")
    ts = neural.TrainStep(p, cfg)
    tok = torch.as_tensor(GOLD["tokens"], device="cuda")
    lengths = torch.full((tok.shape[0],), tok.shape[1], dtype=torch.int32, device="cuda")
    return ts, tok, lengths


@pytest.mark.parametrize("tied", [False, True])
def test_parameter_gradients_match_reference(tied):
    tag = "tied" if tied else "untied"
    ts, tok, lengths = _step(tied)
    loss, grads = ts.loss_and_grads(tok, lengths)
    assert torch.isfinite(loss)
    for k, g in zip(ts.params.tensors, grads):
        want = GOLD[f"{tag}.grad.{k}"]
        got = g.double().cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=FP32, atol=FP32 * np.abs(want).max() + 1e-12,
                                   err_msg=k)


@pytest.mark.parametrize("tied", [False, True])
def test_one_train_step_matches_reference(tied):
    tag = "tied" if tied else "untied"
    ts, tok, lengths = _step(tied)
    ts.step(tok, lengths)
    torch.cuda.synchronize()
    for k, x in ts.params.tensors.items():
        want = GOLD[f"{tag}.step1.{k}"]
        g = GOLD[f"{tag}.grad.{k}"]
        # the first bias-corrected Adam step moves each element by lr * g/|g|:
        # compare where the gradient is not at rounding level
        sure = np.abs(g) > 1e-3 * np.abs(g).max()
        got = x.detach().double().cpu().numpy()
        np.testing.assert_allclose(got[sure], want[sure], rtol=0, atol=1e-6, err_msg=k)


def test_training_reduces_the_loss_bf16():
    dims = GrammarDims(256, 256, 64)
    p = neural.init_params(dims, 64, 0, device="cuda")
    ts = neural.TrainStep(p, neural.TrainConfig(gemm_dtype="bf16", lr=0.01))
    g = torch.Generator(device="cuda").manual_seed(0)
    tok = torch.randint(0, 16, (8, 12), device="cuda", generator=g)  # a skewed corpus
    lengths = torch.full((8,), 12, dtype=torch.int32, device="cuda")
    losses = [float(ts.step(tok, lengths)) for _ in range(15)]
    assert all(np.isfinite(losses))
    assert losses[-1] < losses[0] - 1.0


@pytest.mark.parametrize("rows,cols,d", [(6, 11, 16), (1, 6, 16), (256, 512, 64), (300, 700, 96),
                                         (1024, 2048, 512)])
@pytest.mark.parametrize("gemm_dtype,tol", [("fp32", 1e-5), ("tf32", 2e-3)])
def test_score_table_on_the_engine(rows, cols, d, gemm_dtype, tol):
    """log_softmax(A B^T) and its backward through fi_param_scores(_backward)
    (tcgen05 GEMM + row passes) against float64 torch."""
    g = torch.Generator(device="cuda").manual_seed(rows + cols + d)
    A = torch.randn(rows, d, device="cuda", generator=g) / d ** 0.25
    B = torch.randn(cols, d, device="cuda", generator=g) / d ** 0.25
    up = torch.randn(rows, cols, device="cuda", generator=g)
    A.requires_grad_(True)
    B.requires_grad_(True)
    lp = neural.score_table(A, B, gemm_dtype)
    (lp * up).sum().backward()
    A64 = A.detach().double().requires_grad_(True)
    B64 = B.detach().double().requires_grad_(True)
    lp64 = torch.log_softmax(A64 @ B64.T, dim=-1)
    (lp64 * up.double()).sum().backward()
    for name, got, want in (("logp", lp.detach(), lp64.detach()), ("dA", A.grad, A64.grad),
                            ("dB", B.grad, B64.grad)):
        err = ((got.double() - want).abs().max() / want.abs().max()).item()
        assert err < tol, f"{name}: {err:.2e}"


def test_realistic_size_gradients_match_reference():
    """|N| = P = 256, V = 64, d = 64 (tests/golden/neural.npz "big.*", the
    reference's forward_grammar + inside_backward + backward_params): the
    GPU step's tables and parameter gradients in fp32 mode."""
    dims = GrammarDims(256, 256, 64)
    ts = neural.TrainStep(neural.init_params(dims, 64, SEED, device="cuda"),
                          neural.TrainConfig(gemm_dtype="fp32"))
    with torch.no_grad():
        tabs = ts.tables()
    for name, t in zip(("log_root", "log_left", "log_right", "log_emit"), tabs):
        want = GOLD[f"big.{name}"]
        np.testing.assert_allclose(t.double().cpu().numpy(), want, rtol=FP32,
                                   atol=FP32 * np.abs(want).max(), err_msg=name)
    tok = torch.as_tensor(GOLD["big.tokens"], device="cuda")
    lengths = torch.full((tok.shape[0],), tok.shape[1], dtype=torch.int32, device="cuda")
    loss, grads = ts.loss_and_grads(tok, lengths)
    for k, gr in zip(ts.params.tensors, grads):
        want = GOLD[f"big.grad.{k}"]
        got = gr.double().cpu().numpy()
        np.testing.assert_allclose(got, want, rtol=FP32, atol=FP32 * np.abs(want).max() + 1e-12,
                                   err_msg=k)
