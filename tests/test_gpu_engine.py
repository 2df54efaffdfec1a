"""GPU tests of the reference-facing engine and of full-size properties.

* the reference's golden vectors (tests/golden/golden.npz, produced by the
  reference itself) through inside_b200 / inside_backward_b200 /
  corpus_log_likelihood — closed forms, brute force, chart layout,
  gradients, marginals, the 512-symbol and deep-log-space cases, and the
  SURVEY configs' log Z;
* at BASELINE config 3 (N=P=4096, l=40, B=64) size-independent identities
  that must hold for any correct inside/outside pass.
"""

import math

import numpy as np
import pytest
import torch

from paper_2310_14997_b200 import engine
from paper_2310_14997_b200.grammar import GrammarDims, SimpleGrammar, random_grammar
from paper_2310_14997_b200.ops import inside

pytestmark = pytest.mark.gpu
GOLD = np.load(__file__.replace("test_gpu_engine.py", "golden/golden.npz"))
FP32 = 1e-4   # north-star tolerance of the fp32 mode
BF16 = 2e-3


def g1():
    h = math.log(0.5)
    return SimpleGrammar(GrammarDims(1, 1, 1), np.array([0.0]), np.array([[h, h]]),
                         np.array([[h, h]]), np.array([[0.0]]))


@pytest.mark.parametrize("l,want", [(2, 0.25), (3, 0.125), (4, 0.078125)])
def test_g1_closed_form(l, want):
    chart = engine.inside_b200(g1(), np.zeros(l, dtype=np.int64))
    assert chart.log_z == pytest.approx(math.log(want), rel=FP32)
    assert np.all(chart.o[1][:, :1] == -np.inf)          # chart masking (test_inside.py:144-149)
    assert np.all(chart.o[2][:, 1:] == -np.inf)


def test_g1_marginals_and_ppl():
    g = g1()
    toks = np.zeros(3, dtype=np.int64)
    _, marg = engine.inside_backward_b200(g, toks, engine.inside_b200(g, toks))
    np.testing.assert_allclose([marg.span(0, 2), marg.span(1, 3), marg.span(0, 3)],
                               GOLD["g1_mu_xxx"], atol=1e-5)
    _, ppl = engine.corpus_log_likelihood(g, [np.zeros(2, dtype=np.int64)])
    assert ppl == pytest.approx(2.0, rel=FP32)


def _rand(k):
    pre = f"rand{k}_"
    n, p, v, _ = (int(x) for x in GOLD["rand_meta"][k])
    g = SimpleGrammar(GrammarDims(n, p, v), GOLD[pre + "root"], GOLD[pre + "left"],
                      GOLD[pre + "right"], GOLD[pre + "emit"])
    return g, GOLD[pre + "tokens"], pre


@pytest.mark.parametrize("k", range(0, 40, 3))
def test_reference_instances_logz_grads_marginals(k):
    g, toks, pre = _rand(k)
    chart = engine.inside_b200(g, toks)
    assert chart.log_z == pytest.approx(float(GOLD[pre + "logz"]), rel=FP32, abs=1e-6)
    assert chart.log_z == pytest.approx(float(GOLD[pre + "brute"]), rel=FP32, abs=1e-6)
    grad, marg = engine.inside_backward_b200(g, toks, chart)
    for name in ("d_root", "d_left", "d_right", "d_emit"):
        want = GOLD[pre + name]
        got = getattr(grad, name)
        np.testing.assert_allclose(got, want, rtol=FP32, atol=FP32 * np.abs(want).max(),
                                   err_msg=name)
    mu = np.concatenate([m for m in marg.mu[2:]])
    np.testing.assert_allclose(mu, GOLD[pre + "mu"], atol=1e-5)
    assert grad.d_root.sum() == pytest.approx(1.0, abs=1e-5)   # test_backward.py:61-66


def test_chart_matches_reference_chart():
    g = random_grammar(GrammarDims(3, 4, 5), seed=2)
    chart = engine.inside_b200(g, np.array([1, 3, 0, 2, 4]))
    for w in range(1, 6):
        np.testing.assert_allclose(chart.o[w], GOLD[f"chart_o{w}"], rtol=FP32, atol=1e-5)
    for w in range(1, 5):
        np.testing.assert_allclose(chart.a[w], GOLD[f"chart_a{w}"], rtol=FP32, atol=1e-5)
        np.testing.assert_allclose(chart.b[w], GOLD[f"chart_b{w}"], rtol=FP32, atol=1e-5)


@pytest.mark.parametrize("dtype,tol", [("fp32", FP32), ("bf16", BF16)])
def test_512_symbol_case(dtype, tol):
    g = random_grammar(GrammarDims(256, 256, 64), seed=42)
    got = engine.batched_inside(g, list(GOLD["c2_tokens"]), gemm_dtype=dtype)
    np.testing.assert_allclose(got, GOLD["c2_logz"], rtol=tol)


def test_deep_log_space_stability():
    g = random_grammar(GrammarDims(6, 6, 50), seed=13, concentration=0.3)
    chart = engine.inside_b200(g, GOLD["deep_tokens"])
    assert chart.log_z < -400 and np.isfinite(chart.log_z)
    assert chart.log_z == pytest.approx(float(GOLD["deep_logz"]), rel=FP32)


def test_config1_perplexity():
    g = random_grammar(GrammarDims(64, 64, 64), seed=0)
    toks = list(np.random.default_rng(1).integers(0, 64, (8, 20)))
    lls, ppl = engine.corpus_log_likelihood(g, toks)
    np.testing.assert_allclose(lls, GOLD["cfg1_logz"], rtol=FP32)
    assert ppl == pytest.approx(82.9280131100, rel=FP32)


@pytest.mark.parametrize("n,l", [(1024, 30), (4096, 40)])
@pytest.mark.parametrize("dtype,tol", [("fp32", FP32), ("bf16", BF16), ("tf32", BF16)])
def test_survey_config_log_z(n, l, dtype, tol):
    g = random_grammar(GrammarDims(n, n, 64), seed=0)
    t = np.random.default_rng(1).integers(0, 64, (1, l))
    got = engine.batched_inside(g, list(t), gemm_dtype=dtype)
    assert got[0] == pytest.approx(float(GOLD[f"cfg_n{n}_l{l}_logz0"]), rel=tol)


def test_medium_batch_gradients_through_op():
    """Variable-length batch through the torch op vs the reference's summed grads."""
    g = random_grammar(GrammarDims(16, 12, 10), seed=31)
    lens = GOLD["med_lens"]
    toks = np.split(GOLD["med_tokens"], np.cumsum(lens)[:-1])
    l = int(lens.max())
    dg = engine.DeviceGrammar(g)
    tok = torch.zeros(len(lens), l, dtype=torch.long, device="cuda")
    for b, t in enumerate(toks):
        tok[b, :len(t)] = torch.as_tensor(t)
    L, R, root = (t.clone().requires_grad_(True) for t in (dg.L, dg.R, dg.root))
    un = dg.unary(tok).requires_grad_(True)
    lz = inside(L, R, root, un, torch.tensor(lens, dtype=torch.int32, device="cuda"),
                gemm_dtype="fp32")
    lz.sum().backward()
    np.testing.assert_allclose(lz.detach().cpu().numpy(), GOLD["med_logz"], rtol=FP32)
    for t, name in ((L, "d_left"), (R, "d_right"), (root, "d_root")):
        want = GOLD["med_" + name]
        np.testing.assert_allclose(t.grad.double().cpu().numpy(), want, rtol=FP32,
                                   atol=FP32 * np.abs(want).max(), err_msg=name)


def test_zero_probability_sentence_raises():
    # emission of token 1 impossible for the only preterminal -> log_z = -inf
    g = SimpleGrammar(GrammarDims(1, 1, 2), np.array([0.0]),
                      np.log([[0.5, 0.5]]), np.log([[0.5, 0.5]]), np.array([[0.0, -np.inf]]))
    toks = np.array([0, 1])
    chart = engine.inside_b200(g, toks)
    assert chart.log_z == -np.inf
    with pytest.raises(engine.InsideError, match="zero-probability"):
        engine.inside_backward_b200(g, toks, chart)


@pytest.fixture(scope="module")
def config3():
    n, B, l = 4096, 64, 40
    g = random_grammar(GrammarDims(n, n, 64), seed=0)
    tok = torch.as_tensor(np.random.default_rng(1).integers(0, 64, (B, l)), device="cuda")
    dg = engine.DeviceGrammar(g)
    return g, dg, tok, B, l


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_config3_identities(config3, dtype):
    """Outside-pass identities at full size: every derivation uses the root
    once, every token has exactly one preterminal, and each binary node has
    one left and one right child."""
    g, dg, tok, B, l = config3
    L, R, root = (t.clone().requires_grad_(True) for t in (dg.L, dg.R, dg.root))
    un = dg.unary(tok).requires_grad_(True)
    lengths = torch.full((B,), l, dtype=torch.int32, device="cuda")
    gvec = torch.linspace(-1.0, 2.0, B, device="cuda")
    lz = inside(L, R, root, un, lengths, gemm_dtype=dtype)
    (lz * gvec).sum().backward()
    tol = 2e-3 if dtype == "bf16" else 1e-4
    gs = gvec.double().cpu().numpy()
    assert torch.isfinite(lz).all()
    assert root.grad.double().sum().item() == pytest.approx(gs.sum(), rel=tol, abs=tol)
    per_tok = un.grad.double().sum(-1).cpu().numpy()                # (B, l)
    np.testing.assert_allclose(per_tok, np.repeat(gs[:, None], l, 1), rtol=tol, atol=tol)
    rows_l = L.grad.double().sum(1).cpu().numpy()
    rows_r = R.grad.double().sum(1).cpu().numpy()
    np.testing.assert_allclose(rows_l, rows_r, rtol=tol, atol=tol * np.abs(rows_l).max())
    assert rows_l.sum() == pytest.approx(gs.sum() * (l - 1), rel=tol)


def test_config3_log_z_vs_oracle(config3):
    from oracle import flashinside_oracle as O
    g, dg, tok, B, l = config3
    lengths = torch.full((B,), l, dtype=torch.int32, device="cuda")
    with torch.no_grad():
        lz = inside(dg.L, dg.R, dg.root, dg.unary(tok), lengths, gemm_dtype="fp32")
    t = tok[:2].cpu().numpy()
    want = O.inside_batch(g.log_left, g.log_right, g.log_root,
                          O.unary_from_tokens(np.asarray(g.log_emit), t, l), np.full(2, l),
                          backward=False)["log_z"]
    np.testing.assert_allclose(lz[:2].cpu().numpy(), want, rtol=FP32)
    assert want[0] == pytest.approx(float(GOLD["cfg_n4096_l40_logz0"]), abs=1e-9)


def test_marginals_64_symbols_against_oracle():
    """MarginalTable of a 64-symbol grammar (the vectorised export path)
    against the float64 oracle's go[w][:, :N] (inside.py:425-430)."""
    from oracle import flashinside_oracle as O
    g = random_grammar(GrammarDims(64, 64, 30), seed=5)
    toks = np.random.default_rng(6).integers(0, 30, 12)
    chart = engine.inside_b200(g, toks)
    _, marg = engine.inside_backward_b200(g, toks, chart)
    L, R = np.asarray(g.log_left), np.asarray(g.log_right)
    unary = np.asarray(g.log_emit)[:, toks].T
    ch = O.inside_sentence(L, R, np.asarray(g.log_root), unary)
    *_, go = O.backward_sentence(L, R, np.asarray(g.log_root), ch)
    want = O.marginals_sentence(ch, go)
    for w in range(2, toks.size + 1):
        np.testing.assert_allclose(marg.mu_sym[w], want[w], rtol=FP32, atol=1e-6,
                                   err_msg=f"w={w}")
        np.testing.assert_allclose(marg.mu[w], want[w].sum(axis=1), rtol=FP32, atol=1e-6)
