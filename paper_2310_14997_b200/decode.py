"""Tree decoders and bracketing F1 on the B200 engine.

Mirrors /root/reference/pkg/src/flashpcfg/parse.py:

* ``mbr_decode_batch``  ``mbr_decode`` (parse.py:98-131) over the span
  posteriors of ``inside_backward`` (inside.py:425-430), for a whole batch
  of sentences: one forward with the chart kept, one backward, the span
  masses (``fi_span_marginals``) and a batched CKY (``fi_mbr_decode``) all
  on the GPU; the host only reads the trees off the split tables.
* ``viterbi_decode_batch``  ``viterbi_decode`` (parse.py:33-95): the inside
  recursion in the (max, +) semiring -- tropical projections on the CUDA
  cores, a max-over-splits kernel and a per-sentence device backtrack
  (``fi_viterbi``); ``tree_log_prob`` (parse.py:134-158) rescoring on the host.
* ``sentence_f1``       parse.py:161-183 (trivial spans removed).

Ties prefer the smallest split point, as in the reference.  The engine works
in fp32 (``gemm_dtype="fp32"`` by default here: decoding compares sums of
posteriors, so near-ties are decided at fp32 resolution).
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .engine import DeviceGrammar, InsideError, _prepare
from .ops import _p, _stream, inside_bwd, inside_fwd

Span = tuple[int, int]


class ParseError(Exception):
    """Decoding failure (parse.py:28-29)."""


def _filter_trivial(spans, length: int) -> frozenset:
    return frozenset((i, j) for (i, j) in spans if j - i >= 2 and not (i == 0 and j == length))


def sentence_f1(pred, gold, length: int) -> float:
    """Unlabeled span F1 without the whole-sentence and width-1 spans; two
    empty sets score 1.0, exactly one empty set 0.0 (parse.py:166-183)."""
    p = _filter_trivial(pred, length)
    g = _filter_trivial(gold, length)
    if not p and not g:
        return 1.0
    if not p or not g:
        return 0.0
    hits = len(p & g)
    precision, recall = hits / len(p), hits / len(g)
    if precision + recall == 0.0:
        return 0.0
    return 2.0 * precision * recall / (precision + recall)


def spans_from_splits(split: np.ndarray, length: int) -> frozenset:
    """Internal spans of the tree rooted at (0, length) given split[i, j]."""
    spans: set[Span] = set()
    stack = [(0, length)]
    while stack:
        i, j = stack.pop()
        if j - i < 2:
            continue
        spans.add((i, j))
        k = int(split[i, j])
        stack.append((i, k))
        stack.append((k, j))
    return frozenset(spans)


def _batches(sents, max_batch: int):
    order = sorted(range(len(sents)), key=lambda k: -sents[k].size)
    for s in range(0, len(order), max_batch):
        yield order[s:s + max_batch]


def mbr_decode_batch(g, sentences, gemm_dtype: str = "fp32", dg: DeviceGrammar | None = None,
                     max_batch: int = 64, return_mass: bool = False):
    """MBR trees (frozensets of internal spans, root included) of every sentence.

    Raises InsideError naming the sentence if one has zero probability (the
    reference's inside_backward condition, inside.py:392-393)."""
    sents = [_prepare(g, s) for s in sentences]
    dg = dg or DeviceGrammar(g)
    lib = _lib.load()
    out: list[frozenset | None] = [None] * len(sents)
    masses: list = [None] * len(sents)
    n_nt, n_pt = g.dims.n_nt, g.dims.n_pt
    with torch.no_grad():
        for idx in _batches(sents, max_batch):
            B = len(idx)
            lmax = max(sents[k].size for k in idx)
            tok = torch.zeros(B, lmax, dtype=torch.long, device=dg.device)
            for r, k in enumerate(idx):
                tok[r, :sents[k].size] = torch.as_tensor(sents[k])
            lens = torch.tensor([sents[k].size for k in idx], dtype=torch.int32, device=dg.device)
            unary = dg.unary(tok)
            log_z, ws = inside_fwd(dg.L, dg.R, dg.root, unary, lens, gemm_dtype, True)
            lz = log_z.cpu().numpy()
            for r, k in enumerate(idx):
                if not np.isfinite(lz[r]):
                    raise InsideError(f"sentence {k}: zero-probability sentence; no parse")
            ones = torch.ones(B, dtype=torch.float32, device=dg.device)
            inside_bwd(ones, dg.L, dg.R, dg.root, unary, lens, log_z, ws, gemm_dtype, True)
            shape = _lib.shape(n_nt, n_pt, B, lmax, gemm_dtype, True)
            nrows = int(_lib.chart_layout(shape).rows) - B * lmax
            mass = torch.empty(max(nrows, 1), dtype=torch.float32, device=dg.device)
            score = torch.empty(B, lmax, lmax + 1, dtype=torch.float32, device=dg.device)
            split = torch.zeros(B, lmax, lmax + 1, dtype=torch.int32, device=dg.device)
            st = _stream(dg.device)
            _lib.check(lib.fi_span_marginals(ctypes.byref(shape), _p(lens), _p(ones), _p(mass),
                                             _p(ws), st))
            _lib.check(lib.fi_mbr_decode(ctypes.byref(shape), _p(lens), _p(mass), _p(score),
                                         _p(split), st))
            sp = split.cpu().numpy()
            m_np = mass.double().cpu().numpy() if return_mass else None
            for r, k in enumerate(idx):
                l = sents[k].size
                out[k] = spans_from_splits(sp[r], l)
                if return_mass:  # mu[i, j] for the sentence, as MarginalTable.span
                    mu = np.zeros((l + 1, l + 1))
                    base = 0
                    for w in range(2, lmax + 1):
                        n_w = lmax - w + 1
                        if w <= l:
                            mu[np.arange(l - w + 1), np.arange(l - w + 1) + w] = \
                                m_np[base + r * n_w: base + r * n_w + l - w + 1]
                        base += B * n_w
                    masses[k] = mu
    return (out, masses) if return_mass else out


def mbr_score(mu: np.ndarray, spans) -> float:
    """Total posterior mass of a tree's internal spans (the MBR objective)."""
    return float(sum(mu[i, j] for (i, j) in spans))


# ------------------------------------------------------------------ Viterbi
def viterbi_decode_batch(g, sentences, dg: DeviceGrammar | None = None, max_batch: int = 64):
    """Best derivation of every sentence (viterbi_decode, parse.py:33-95).

    Returns a list of dicts {"spans": frozenset, "labels": {(i, j): "NT<a>"},
    "leaf_labels": ("PT<t>", ...), "log_prob": float}.  The (max, +) chart,
    the tropical projections and the backtrack all run on the GPU."""
    sents = [_prepare(g, s) for s in sentences]
    dg = dg or DeviceGrammar(g)
    lib = _lib.load()
    n_nt, n_pt = g.dims.n_nt, g.dims.n_pt
    out: list = [None] * len(sents)
    with torch.no_grad():
        for idx in _batches(sents, max_batch):
            B = len(idx)
            lmax = max(sents[k].size for k in idx)
            tok = torch.zeros(B, lmax, dtype=torch.long, device=dg.device)
            for r, k in enumerate(idx):
                tok[r, :sents[k].size] = torch.as_tensor(sents[k])
            lens = torch.tensor([sents[k].size for k in idx], dtype=torch.int32, device=dg.device)
            unary = dg.unary(tok)
            shape = _lib.shape(n_nt, n_pt, B, lmax, "fp32", False)
            lay = _lib.chart_layout(shape)
            rows, np_ = int(lay.rows), int(lay.np)
            va, vb, vo = (torch.empty(rows, np_, dtype=torch.float32, device=dg.device)
                          for _ in range(3))
            nodes = torch.zeros(B, 2 * lmax, 3, dtype=torch.int32, device=dg.device)
            best = torch.empty(B, dtype=torch.float32, device=dg.device)
            _lib.check(lib.fi_viterbi(ctypes.byref(shape), _p(dg.L), _p(dg.R), _p(dg.root),
                                      _p(unary), _p(lens), _p(va), _p(vb), _p(vo), _p(nodes),
                                      _p(best), _stream(dg.device)))
            nd = nodes.cpu().numpy()
            bs = best.double().cpu().numpy()
            for r, k in enumerate(idx):
                l = sents[k].size
                if not np.isfinite(bs[r]):
                    raise ParseError(f"sentence {k}: no parse with positive probability")
                spans, labels, leaves = set(), {}, [""] * l
                for i, j, sym in nd[r, :2 * l - 1]:
                    if j - i == 1:
                        leaves[int(i)] = f"PT{int(sym)}"
                    else:
                        spans.add((int(i), int(j)))
                        labels[(int(i), int(j))] = f"NT{int(sym)}"
                out[k] = {"spans": frozenset(spans), "labels": labels,
                          "leaf_labels": tuple(leaves), "log_prob": float(bs[r])}
    return out


def tree_log_prob(g, tokens, tree: dict) -> float:
    """Log probability of a labelled derivation (parse.py:134-158), float64 on the host."""
    toks = np.asarray(tokens, dtype=np.int64)
    n_nt = g.dims.n_nt
    spans = tree["spans"]
    l = toks.size

    def sym_of(i, j):
        if j - i == 1:
            return n_nt + int(tree["leaf_labels"][i][2:])
        return int(tree["labels"][(i, j)][2:])

    def covered(i, j):
        return j - i == 1 or (i, j) in spans

    total = g.log_root[sym_of(0, l)]
    for (i, j) in spans:
        k = next(k for k in range(i + 1, j) if covered(i, k) and covered(k, j))
        parent = sym_of(i, j)
        total += g.log_left[parent, sym_of(i, k)] + g.log_right[parent, sym_of(k, j)]
    for i, tok in enumerate(toks):
        total += g.log_emit[sym_of(i, i + 1) - n_nt, tok]
    return float(total)
