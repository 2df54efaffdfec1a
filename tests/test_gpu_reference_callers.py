"""The drop-in, proven through the reference's OWN code: the unmodified
flashpcfg package (installed into baseline/_ref by the recipe in DESIGN.md
§7; it travels to the GPU box with the repo snapshot) with the B200 engine
registered into its ENGINES dict, driven by its own callers:

* ``corpus_log_likelihood(engine="b200")``   inside.py:555-578
* ``inside_backward`` on a b200 chart         inside.py:375-447 (bitwise
                                              o[1] check at :390)
* ``corpus_f1(decoder="mbr", engine="b200")`` parse.py:267-316
* ``train(TrainConfig(engine="b200"))``       train.py:180, :209-214

each against the same call with the reference's own engine ("flash").
Skipped when baseline/_ref is absent (the package is not vendored)."""

import sys
from pathlib import Path

import numpy as np
import pytest

REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not (REF / "flashpcfg").is_dir(),
                                 reason="reference package not installed in baseline/_ref")]


@pytest.fixture(scope="module")
def ref():
    sys.path.insert(0, str(REF))
    import flashpcfg.inside as rinside
    import flashpcfg.parse as rparse
    import flashpcfg.train as rtrain
    from flashpcfg import data as rdata
    from flashpcfg.grammar import GrammarDims, random_grammar
    from paper_2310_14997_b200 import engine
    engine.register(rinside.ENGINES)   # the reference's own registry (inside.py:343-348)
    assert rinside.ENGINES["b200"] is engine.inside_b200
    return dict(inside=rinside, parse=rparse, train=rtrain, data=rdata, GrammarDims=GrammarDims,
                random_grammar=random_grammar, engine=engine)


def _corpus(V, n, lo, hi, seed):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, V, size=int(rng.integers(lo, hi + 1))) for _ in range(n)]


def test_corpus_log_likelihood_through_the_registry(ref):
    g = ref["random_grammar"](ref["GrammarDims"](48, 40, 30), seed=4)
    sents = _corpus(30, 12, 2, 14, 5)
    lls_b, ppl_b = ref["inside"].corpus_log_likelihood(g, sents, engine="b200")
    lls_f, ppl_f = ref["inside"].corpus_log_likelihood(g, sents, engine="flash")
    np.testing.assert_allclose(lls_b, lls_f, rtol=1e-4)
    assert ppl_b == pytest.approx(ppl_f, rel=1e-4)


def test_reference_backward_accepts_the_b200_chart(ref):
    g = ref["random_grammar"](ref["GrammarDims"](24, 20, 16), seed=7)
    toks = np.array([3, 1, 4, 1, 5, 9, 2, 6, 5, 3, 5])
    chart_b = ref["inside"].ENGINES["b200"](g, toks)
    chart_f = ref["inside"].inside_flash(g, toks)
    assert chart_b.log_z == pytest.approx(chart_f.log_z, rel=1e-4)
    gb, mb = ref["inside"].inside_backward(g, toks, chart_b)   # the reference's own backward
    gf, mf = ref["inside"].inside_backward(g, toks, chart_f)
    for name in ("d_root", "d_left", "d_right", "d_emit"):
        want = getattr(gf, name)
        np.testing.assert_allclose(getattr(gb, name), want, rtol=1e-4,
                                   atol=1e-4 * np.abs(want).max(), err_msg=name)
    for w in range(2, len(toks) + 1):
        np.testing.assert_allclose(mb.mu[w], mf.mu[w], rtol=1e-4, atol=1e-6)
    # and our own backward on the same chart returns the reference's GrammarGrad
    g2, m2 = ref["engine"].inside_backward_b200(g, toks, chart_b)
    for name in ("d_root", "d_left", "d_right", "d_emit"):
        want = getattr(gf, name)
        np.testing.assert_allclose(getattr(g2, name), want, rtol=1e-4,
                                   atol=1e-4 * np.abs(want).max(), err_msg=name)


def test_backward_refuses_a_chart_of_another_grammar(ref):
    dims = ref["GrammarDims"](8, 6, 10)
    g1 = ref["random_grammar"](dims, seed=1)
    g2 = ref["random_grammar"](dims, seed=2)
    toks = np.array([1, 2, 3, 4])
    chart = ref["inside"].ENGINES["b200"](g1, toks)
    with pytest.raises(ref["inside"].InsideError, match="not produced from this grammar"):
        ref["inside"].inside_backward(g2, toks, chart)
    with pytest.raises(ref["engine"].InsideError, match="not produced from this grammar"):
        ref["engine"].inside_backward_b200(g2, toks, chart)


def test_corpus_f1_mbr_through_the_registry(ref):
    P = ref["parse"]
    g = ref["random_grammar"](ref["GrammarDims"](16, 12, 8), seed=3)
    rng = np.random.default_rng(8)
    bank = []
    for k in range(6):
        l = int(rng.integers(3, 10))
        toks = tuple(f"w{int(t)}" for t in rng.integers(0, 8, l))
        spans = frozenset({(0, l)} | {(i, i + 2) for i in range(0, l - 1, 2)})
        bank.append(P.GoldAnnotation(toks, ("X",) * l, spans, (False,) * l))

    def encode(words):
        return [int(w[1:]) for w in words]
    fb = P.corpus_f1(g, bank, encode, decoder="mbr", engine="b200")
    ff = P.corpus_f1(g, bank, encode, decoder="mbr", engine="flash")
    assert fb.mean_f1 == pytest.approx(ff.mean_f1, abs=1e-12)
    assert [r[:2] for r in fb.rows] == [r[:2] for r in ff.rows]


@pytest.mark.parametrize("parameterization", ["direct", "neural"])
def test_reference_training_loop_on_the_b200_engine(ref, parameterization):
    T, D = ref["train"], ref["data"]
    train_s = _corpus(12, 10, 3, 8, 11)
    dev_s = _corpus(12, 4, 3, 8, 12)
    mk = lambda s: D.Corpus(s, [[]] * len(s))  # noqa: E731
    runs = {}
    for eng in ("b200", "flash"):
        cfg = T.TrainConfig(parameterization=parameterization, n_nt=10, n_pt=8, d=16,
                            max_epochs=2, batch_cap=16, eval_every=3, seed=0, engine=eng,
                            vocab_size=12, lr=0.01)
        runs[eng] = T.train(cfg, mk(train_s), mk(dev_s))
    lb = np.array([l for _, l in runs["b200"].log.steps])
    lf = np.array([l for _, l in runs["flash"].log.steps])
    assert len(lb) == len(lf) > 3
    np.testing.assert_allclose(lb, lf, rtol=1e-4)
    eb = np.array([p for _, p in runs["b200"].log.evals])
    ef = np.array([p for _, p in runs["flash"].log.evals])
    np.testing.assert_allclose(eb, ef, rtol=1e-4)
