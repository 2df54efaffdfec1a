"""Golden vectors for the decoders, from the REFERENCE (run where
/root/reference exists):

    python tests/golden/make_golden_decode.py

Writes tests/golden/decode.npz: for seeded random grammars and sentences,
the reference's span marginals (inside_backward -> MarginalTable.mu), its
MBR tree (mbr_decode, parse.py:98-131), its Viterbi tree with the tree's
log probability (viterbi_decode / tree_log_prob, parse.py:33-95, :134-158),
and sentence F1 values (parse.py:161-183).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from flashpcfg.grammar import GrammarDims, random_grammar  # noqa: E402
from flashpcfg.inside import inside_backward, inside_flash  # noqa: E402
from flashpcfg.parse import (mbr_decode, sentence_f1, tree_log_prob,  # noqa: E402
                             viterbi_decode)

OUT = Path(__file__).resolve().parent / "decode.npz"


def spans_arr(spans):
    return np.array(sorted(spans), dtype=np.int64).reshape(-1, 2)


def main():
    gold = {}
    rng = np.random.default_rng(23)
    cases = []
    for k in range(12):
        n_nt = int(rng.integers(2, 9))
        n_pt = int(rng.integers(2, 9))
        V = int(rng.integers(3, 12))
        gseed = int(rng.integers(0, 10_000))
        conc = float(rng.choice([0.3, 1.0]))
        g = random_grammar(GrammarDims(n_nt, n_pt, V), seed=gseed, concentration=conc)
        l = int(rng.integers(2, 14))
        toks = rng.integers(0, V, size=l)
        chart = inside_flash(g, toks)
        _, marg = inside_backward(g, toks, chart)
        mbr = mbr_decode(marg)
        vit = viterbi_decode(g, toks)
        pre = f"c{k}_"
        gold[pre + "meta"] = np.array([n_nt, n_pt, V, gseed, l])
        gold[pre + "conc"] = np.array(conc)
        gold[pre + "tokens"] = toks
        mu = np.zeros((l + 1, l + 1))
        for w in range(2, l + 1):
            for i in range(l - w + 1):
                mu[i, i + w] = marg.span(i, i + w)
        gold[pre + "mu"] = mu
        gold[pre + "mbr"] = spans_arr(mbr.spans)
        gold[pre + "vit"] = spans_arr(vit.spans)
        gold[pre + "vit_logp"] = np.array(tree_log_prob(g, toks, vit))
        gold[pre + "f1_mbr_vs_vit"] = np.array(sentence_f1(mbr.spans, vit.spans, l))
        cases.append(k)
    # realistic sizes (|N| = 256 .. 1024): the decoders at the op's scale
    big = [(256, 256, 64, 20, 1.0), (256, 256, 64, 24, 0.3), (512, 512, 64, 16, 1.0),
           (1024, 1024, 64, 12, 1.0), (1024, 1024, 64, 10, 0.3)]
    for j, (n_nt, n_pt, V, l, conc) in enumerate(big):
        k = len(cases)
        gseed = 1000 + j
        g = random_grammar(GrammarDims(n_nt, n_pt, V), seed=gseed, concentration=conc)
        toks = np.random.default_rng(gseed + 1).integers(0, V, size=l)
        chart = inside_flash(g, toks)
        _, marg = inside_backward(g, toks, chart)
        mbr = mbr_decode(marg)
        vit = viterbi_decode(g, toks)
        pre = f"c{k}_"
        gold[pre + "meta"] = np.array([n_nt, n_pt, V, gseed, l])
        gold[pre + "conc"] = np.array(conc)
        gold[pre + "tokens"] = toks
        mu = np.zeros((l + 1, l + 1))
        for w in range(2, l + 1):
            for i in range(l - w + 1):
                mu[i, i + w] = marg.span(i, i + w)
        gold[pre + "mu"] = mu
        gold[pre + "mbr"] = spans_arr(mbr.spans)
        gold[pre + "vit"] = spans_arr(vit.spans)
        gold[pre + "vit_logp"] = np.array(tree_log_prob(g, toks, vit))
        gold[pre + "f1_mbr_vs_vit"] = np.array(sentence_f1(mbr.spans, vit.spans, l))
        cases.append(k)
    gold["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT, **gold)
    print(f"wrote {OUT} ({len(cases)} cases)")


if __name__ == "__main__":
    main()
