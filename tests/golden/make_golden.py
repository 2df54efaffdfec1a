"""Generate golden vectors from the REFERENCE implementation (run where
/root/reference exists; the GPU box never reads /root/reference).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes tests/golden/golden.npz.  Every value comes from the reference's own
code path (inside_flash / inside_reference / inside_backward /
brute_force_logprob / corpus_log_likelihood), on the fixtures its own tests
use (pkg/tests/conftest.py, test_inside.py, test_backward.py,
test_acceptance.py) and on the SURVEY configs.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

from conftest import make_g1, random_instance  # noqa: E402  (reference fixtures)
from flashpcfg.grammar import GrammarDims, random_grammar  # noqa: E402
from flashpcfg.inside import (  # noqa: E402
    brute_force_logprob, corpus_log_likelihood, inside_backward, inside_flash,
    inside_reference)

OUT = Path(__file__).resolve().parent / "golden.npz"


def main():
    gold = {}
    # G1 closed form (conftest.py:11-24, test_inside.py:61-74)
    g1 = make_g1()
    for l in (2, 3, 4):
        gold[f"g1_logz_{l}"] = np.array(inside_flash(g1, np.zeros(l, dtype=np.int64)).log_z)
    _, marg = inside_backward(g1, np.zeros(3, dtype=np.int64),
                              inside_flash(g1, np.zeros(3, dtype=np.int64)))
    gold["g1_mu_xxx"] = np.array([marg.span(0, 2), marg.span(1, 3), marg.span(0, 3)])
    _, ppl = corpus_log_likelihood(g1, [np.zeros(2, dtype=np.int64)])
    gold["g1_ppl_xx"] = np.array(ppl)

    # random tiny instances: inside_flash, brute force, full GrammarGrad
    rng = np.random.default_rng(17)
    meta = []
    for k in range(40):
        g, toks = random_instance(rng)
        chart = inside_flash(g, toks)
        gr, mg = inside_backward(g, toks, chart)
        d = g.dims
        meta.append((d.n_nt, d.n_pt, d.vocab_size, len(toks)))
        pre = f"rand{k}_"
        gold[pre + "root"] = g.log_root
        gold[pre + "left"] = g.log_left
        gold[pre + "right"] = g.log_right
        gold[pre + "emit"] = g.log_emit
        gold[pre + "tokens"] = toks
        gold[pre + "logz"] = np.array(chart.log_z)
        gold[pre + "brute"] = np.array(brute_force_logprob(g, toks))
        gold[pre + "d_root"] = gr.d_root
        gold[pre + "d_left"] = gr.d_left
        gold[pre + "d_right"] = gr.d_right
        gold[pre + "d_emit"] = gr.d_emit
        gold[pre + "mu"] = np.concatenate([np.asarray(m) for m in mg.mu[2:]])
    gold["rand_meta"] = np.array(meta)

    # chart-level layout (test_inside.py:101-111)
    g = random_grammar(GrammarDims(3, 4, 5), seed=2)
    toks = np.array([1, 3, 0, 2, 4], dtype=np.int64)
    ref = inside_reference(g, toks)
    for w in range(1, 6):
        gold[f"chart_o{w}"] = ref.o[w]
    for w in range(1, 5):
        gold[f"chart_a{w}"] = ref.a[w]
        gold[f"chart_b{w}"] = ref.b[w]

    # 512-symbol agreement case (test_acceptance.py:73-84), flash only
    g = random_grammar(GrammarDims(256, 256, 64), seed=42)
    rng = np.random.default_rng(7)
    toks = np.stack([rng.integers(0, 64, size=40) for _ in range(20)])
    gold["c2_tokens"] = toks
    gold["c2_logz"] = np.array([inside_flash(g, t).log_z for t in toks])

    # deep log-space stability (test_inside.py:113-124)
    g = random_grammar(GrammarDims(6, 6, 50), seed=13, concentration=0.3)
    toks = np.random.default_rng(1).integers(0, 50, size=120).astype(np.int64)
    gold["deep_tokens"] = toks
    gold["deep_logz"] = np.array(inside_flash(g, toks).log_z)

    # medium gradient case: batch of 3 sentences, summed GrammarGrad
    g = random_grammar(GrammarDims(16, 12, 10), seed=31)
    rng = np.random.default_rng(32)
    lens = [9, 7, 2]
    toks = [rng.integers(0, 10, size=n).astype(np.int64) for n in lens]
    acc = None
    for t in toks:
        gr, _ = inside_backward(g, t, inside_flash(g, t))
        acc = gr if acc is None else acc.add_(gr)
    gold["med_tokens"] = np.concatenate(toks)
    gold["med_lens"] = np.array(lens)
    for name in ("d_root", "d_left", "d_right", "d_emit"):
        gold["med_" + name] = getattr(acc, name)
    gold["med_logz"] = np.array([inside_flash(g, t).log_z for t in toks])

    # SURVEY configs: random_grammar(GrammarDims(N,N,64), seed=0), tokens rng(1)
    g = random_grammar(GrammarDims(64, 64, 64), seed=0)
    toks = np.random.default_rng(1).integers(0, 64, (8, 20))
    lls, ppl = corpus_log_likelihood(g, list(toks))
    gold["cfg1_logz"] = np.array(lls)
    gold["cfg1_ppl"] = np.array(ppl)
    # config 2, 3, 4 (|N| = 4096 at l = 10..60) and 5 (|N| = 8192): sentence 0
    for n, l in ((1024, 30), (4096, 40), (4096, 10), (4096, 20), (4096, 30), (4096, 50),
                 (4096, 60), (8192, 40)):
        g = random_grammar(GrammarDims(n, n, 64), seed=0)
        t = np.random.default_rng(1).integers(0, 64, (1, l))[0]
        gold[f"cfg_n{n}_l{l}_logz0"] = np.array(inside_flash(g, t).log_z)

    np.savez_compressed(OUT, **gold)
    print(f"wrote {OUT} ({OUT.stat().st_size / 1e6:.2f} MB, {len(gold)} arrays)")


if __name__ == "__main__":
    main()
