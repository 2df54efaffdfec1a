"""Golden vectors for the grammar parameterisations and the training step,
from the REFERENCE (run where /root/reference exists):

    python tests/golden/make_golden_neural.py

Writes tests/golden/neural.npz: init_params tensors, forward_grammar tables
(neural, tied and direct), backward_params / backward_direct for a grammar
gradient produced by the reference's own inside_backward on a batch, and
the parameters after one reference train step (train.py:201-227 on that
batch: -1/B scaling, global-norm clip 5.0, bias-corrected Adam).
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")

from flashpcfg.grammar import GrammarDims, GrammarGrad  # noqa: E402
from flashpcfg.inside import inside_backward, inside_flash  # noqa: E402
from flashpcfg.neuralparam import (  # noqa: E402
    AdamState, adam_step, backward_direct, backward_params, forward_grammar,
    forward_grammar_direct, init_direct, init_params)
from flashpcfg.train import _clip_grads  # noqa: E402

OUT = Path(__file__).resolve().parent / "neural.npz"
DIMS = (6, 5, 9)   # n_nt, n_pt, vocab
D = 16
SEED = 3


def main():
    dims = GrammarDims(*DIMS)
    gold = {"dims": np.array(DIMS), "d": np.array(D), "seed": np.array(SEED)}
    params = init_params(dims, D, SEED)
    for k, v in params.tensors.items():
        gold["init." + k] = v.copy()
    toks = np.random.default_rng(SEED + 1).integers(0, DIMS[2], size=(4, 7))
    gold["tokens"] = toks
    for tied in (False, True):
        tag = "tied" if tied else "untied"
        g = forward_grammar(params, tied=tied)
        for name in ("log_root", "log_left", "log_right", "log_emit"):
            gold[f"{tag}.{name}"] = getattr(g, name).copy()
        total = GrammarGrad.zeros(dims)
        for row in toks:
            gr, _ = inside_backward(g, row, inside_flash(g, row))
            total.add_(gr)
        total.scale_(-1.0 / len(toks))
        for name in ("d_root", "d_left", "d_right", "d_emit"):
            gold[f"{tag}.gg.{name}"] = getattr(total, name).copy()
        pg = backward_params(params, total, tied=tied)
        for k, v in pg.tensors.items():
            gold[f"{tag}.grad.{k}"] = v.copy()
        # one train step (train.py:215-226): clip then Adam, from fresh params
        p2 = init_params(dims, D, SEED)
        grads = {k: v.copy() for k, v in pg.tensors.items()}
        gold[f"{tag}.clip_norm"] = np.array(_clip_grads(grads, 5.0))
        state = AdamState.zeros(p2.tensors)
        adam_step(p2.tensors, grads, state)
        for k, v in p2.tensors.items():
            gold[f"{tag}.step1.{k}"] = v.copy()
    # direct parameterisation
    dl = init_direct(dims, SEED)
    for k, v in dl.tensors.items():
        gold["direct.init." + k] = v.copy()
    g = forward_grammar_direct(dl)
    total = GrammarGrad.zeros(dims)
    for row in toks:
        gr, _ = inside_backward(g, row, inside_flash(g, row))
        total.add_(gr)
    total.scale_(-1.0 / len(toks))
    for name in ("d_root", "d_left", "d_right", "d_emit"):
        gold[f"direct.gg.{name}"] = getattr(total, name).copy()
    bd = backward_direct(dl, total)
    for k, v in bd.tensors.items():
        gold["direct.grad." + k] = v.copy()
    # realistic size: |N| = P = 256, V = 64, d = 64 (the GPU step's parity at scale)
    bdims = GrammarDims(256, 256, 64)
    bp = init_params(bdims, 64, SEED)
    btoks = np.random.default_rng(SEED + 2).integers(0, 64, size=(4, 10))
    gold["big.tokens"] = btoks
    g = forward_grammar(bp)
    for name in ("log_root", "log_left", "log_right", "log_emit"):
        gold[f"big.{name}"] = getattr(g, name).copy()
    total = GrammarGrad.zeros(bdims)
    for row in btoks:
        gr, _ = inside_backward(g, row, inside_flash(g, row))
        total.add_(gr)
    total.scale_(-1.0 / len(btoks))
    pg = backward_params(bp, total)
    for k, v in pg.tensors.items():
        gold[f"big.grad.{k}"] = v.copy()
    np.savez_compressed(OUT, **gold)
    print(f"wrote {OUT} ({len(gold)} arrays)")


if __name__ == "__main__":
    main()
