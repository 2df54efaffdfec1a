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
