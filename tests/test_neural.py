"""Grammar parameterisations and optimiser (CPU, float64) against golden
vectors produced by the reference's neuralparam.py / train.py
(tests/golden/make_golden_neural.py)."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2310_14997_b200 import neural
from paper_2310_14997_b200.grammar import GrammarDims

GOLD = np.load(Path(__file__).parent / "golden" / "neural.npz")
DIMS = GrammarDims(*(int(x) for x in GOLD["dims"]))
D, SEED = int(GOLD["d"]), int(GOLD["seed"])


def params64():
    return neural.init_params(DIMS, D, SEED, dtype=torch.float64)


def test_init_params_draws_match_reference():
    p = params64()
    for k, v in p.tensors.items():
        np.testing.assert_array_equal(v.numpy(), GOLD["init." + k], err_msg=k)


@pytest.mark.parametrize("tied", [False, True])
def test_grammar_tables_match_forward_grammar(tied):
    tag = "tied" if tied else "untied"
    tabs = neural.grammar_tables_torch(params64(), tied)
    for name, t in zip(("log_root", "log_left", "log_right", "log_emit"), tabs):
        np.testing.assert_allclose(t.numpy(), GOLD[f"{tag}.{name}"], rtol=1e-12, atol=1e-12,
                                   err_msg=name)


@pytest.mark.parametrize("tied", [False, True])
def test_autograd_matches_backward_params(tied):
    """d/dparams of sum(gg * tables) == the reference's manual backward."""
    tag = "tied" if tied else "untied"
    p = params64()
    xs = list(p.tensors.values())
    for x in xs:
        x.requires_grad_(True)
    tabs = neural.grammar_tables_torch(p, tied)
    gg = [torch.tensor(GOLD[f"{tag}.gg.{n}"]) for n in ("d_root", "d_left", "d_right", "d_emit")]
    if tied:  # the reference adds d_left + d_right onto the single left head
        obj = (gg[0] * tabs[0]).sum() + ((gg[1] + gg[2]) * tabs[1]).sum() + (gg[3] * tabs[3]).sum()
    else:
        obj = sum((g * t).sum() for g, t in zip(gg, tabs))
    grads = torch.autograd.grad(obj, xs, allow_unused=True)
    for k, g in zip(p.tensors, grads):
        want = GOLD[f"{tag}.grad.{k}"]
        got = np.zeros_like(want) if g is None else g.numpy()
        np.testing.assert_allclose(got, want, rtol=1e-10, atol=1e-12 * max(1.0, abs(want).max()),
                                   err_msg=k)


@pytest.mark.parametrize("tied", [False, True])
def test_clip_and_adam_step_match_reference(tied):
    tag = "tied" if tied else "untied"
    p = params64()
    grads = {k: torch.tensor(GOLD[f"{tag}.grad.{k}"]) for k in p.tensors}
    norm = neural.clip_grads_(grads, 5.0)
    assert float(norm) == pytest.approx(float(GOLD[f"{tag}.clip_norm"]), rel=1e-12)
    state = neural.AdamState.zeros(p.tensors)
    neural.adam_step(p.tensors, grads, state)
    for k, v in p.tensors.items():
        np.testing.assert_allclose(v.numpy(), GOLD[f"{tag}.step1.{k}"], rtol=1e-12, atol=1e-14,
                                   err_msg=k)


def test_direct_parameterisation_matches_reference():
    dl = neural.init_direct(DIMS, SEED, dtype=torch.float64)
    for k, v in dl.tensors.items():
        np.testing.assert_array_equal(v.numpy(), GOLD["direct.init." + k])
    xs = list(dl.tensors.values())
    for x in xs:
        x.requires_grad_(True)
    tabs = neural.direct_tables(dl)
    gg = [torch.tensor(GOLD[f"direct.gg.{n}"]) for n in ("d_root", "d_left", "d_right", "d_emit")]
    grads = torch.autograd.grad(sum((g * t).sum() for g, t in zip(gg, tabs)), xs)
    for k, g in zip(dl.tensors, grads):
        np.testing.assert_allclose(g.numpy(), GOLD["direct.grad." + k], rtol=1e-10, atol=1e-14)


def test_nonfinite_gradient_is_rejected():
    p = params64()
    grads = {k: torch.zeros_like(v) for k, v in p.tensors.items()}
    grads["u_nt"][0, 0] = float("nan")
    with pytest.raises(neural.ParamError, match="u_nt"):
        neural.adam_step(p.tensors, grads, neural.AdamState.zeros(p.tensors))
    with pytest.raises(neural.ParamError):
        neural.init_params(DIMS, 1)
