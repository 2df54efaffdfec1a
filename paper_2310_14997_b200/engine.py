"""Reference-facing engine API on top of the CUDA op (the drop-in boundary).

The reference's plug-in seam is the name-keyed registry
``ENGINES: dict[str, Callable[[g, tokens, meter], InsideChart]]``
(pkg/src/flashpcfg/inside.py:343-348) plus
``inside_backward(g, tokens, chart) -> (GrammarGrad, MarginalTable)``
(inside.py:375-376).  This module provides, with the same names, argument
meaning and error behaviour:

* ``inside_b200(g, tokens, meter=None)``      an ENGINES entry (one sentence)
* ``inside_backward_b200(g, tokens, chart)``  backward on a b200 chart
* ``ENGINES`` / ``register(registry)``        registry seam
* ``corpus_log_likelihood(g, sentences)``     inside.py:555-578, batched
* ``batched_inside(...)``                     equal-length batches, the way
                                              the training loop feeds it
                                              (train.py:201-218, data.py:161-185)

Grammars may be this package's SimpleGrammar or the reference's own (duck
typed: .dims, .log_root, .log_left, .log_right, .log_emit).  All compute
runs in the sm_100a library; the host only gathers rows and copies.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .grammar import GrammarGrad
from .ops import inside_bwd, inside_fwd, _p, _stream

NEG_INF = float("-inf")
DEFAULT_GEMM_DTYPE = "fp32"  # the strict (1e-4) mode for the reference-facing API


class InsideError(Exception):
    """Invalid input to an inside computation (inside.py:31-32)."""


class AllocMeter:
    """Arena-style allocation accounting (inside.py:35-63), same API.

    Host arrays go through :meth:`alloc` / :meth:`release` as in the
    reference (the exported float64 chart is ``retained``).  The engine's
    device memory is one caller-visible workspace per call (chart + the
    state the backward recomputes from, fi_workspace_bytes): it is counted
    in ``device_retained_bytes``; the engine allocates no device or host
    transients of its own, so ``transient_bytes`` returns to 0 and
    ``peak_transient_bytes`` stays 0 for an engine call."""

    def __init__(self):
        self.transient_bytes = 0
        self.peak_transient_bytes = 0
        self.retained_bytes = 0
        self.device_retained_bytes = 0

    def alloc(self, shape, dtype=np.float64, retained: bool = False) -> np.ndarray:
        arr = np.empty(shape, dtype=dtype)
        if retained:
            self.retained_bytes += arr.nbytes
        else:
            self.transient_bytes += arr.nbytes
            self.peak_transient_bytes = max(self.peak_transient_bytes, self.transient_bytes)
        return arr

    def release(self, arr: np.ndarray) -> None:
        self.transient_bytes -= arr.nbytes

    def device(self, nbytes: int) -> None:
        self.device_retained_bytes += int(nbytes)


@dataclass
class InsideChart:
    """Reference chart layout (inside.py:66-84): o[w] (n_w, n_sym), a[w]/b[w]
    (n_w, N), log_z.  ``_device`` keeps the GPU state for the backward."""

    length: int
    o: list
    a: list
    b: list
    log_z: float
    _device: dict | None = field(default=None, repr=False)

    def beta(self, i: int, j: int) -> np.ndarray:
        return self.o[j - i][i]


@dataclass
class MarginalTable:
    """Span posteriors (inside.py:355-372)."""

    length: int
    mu: list
    mu_sym: list | None = None

    def span(self, i: int, j: int) -> float:
        return float(self.mu[j - i][i])

    def total(self) -> float:
        return float(sum(arr.sum() for arr in self.mu[2:]))


def _prepare(g, tokens) -> np.ndarray:
    """Token validation with the reference's messages (inside.py:113-121)."""
    toks = np.asarray(tokens, dtype=np.int64)
    if toks.ndim != 1 or toks.size < 2:
        raise InsideError(f"need a token sequence of length >= 2, got shape {toks.shape}")
    bad = (toks < 0) | (toks >= g.dims.vocab_size)
    if bad.any():
        raise InsideError(
            f"unknown token id {int(toks[bad][0])} (vocab size {g.dims.vocab_size})")
    return toks


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("the b200 engine needs a CUDA device; there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


class DeviceGrammar:
    """fp32 device copies of a grammar's tables (uploaded once, reused)."""

    def __init__(self, g, device=None):
        dev = device or _device()
        self.g = g
        def up(a):
            return torch.tensor(np.asarray(a, dtype=np.float32), device=dev)
        self.L = up(g.log_left)
        self.R = up(g.log_right)
        self.root = up(g.log_root)
        self.emit = up(g.log_emit)
        self.device = dev

    def unary(self, tokens: torch.Tensor) -> torch.Tensor:
        """unary[b, i, T] = log_emit[T, tokens[b, i]]  (inside.py:296-298)."""
        return self.emit.t()[tokens].contiguous()


_DG_CACHE: list = []  # the last few (grammar, DeviceGrammar) pairs, by identity


def device_grammar(g) -> DeviceGrammar:
    """The device copy of ``g``, uploaded once and reused across per-sentence
    engine calls (the reference's train loop calls the engine once per
    sentence with the same grammar, train.py:208).  Grammars are immutable
    (read-only arrays, grammar.py:56-59), so identity is a sound key; the
    cache holds strong references to at most 2 grammars."""
    dev = _device()
    for gg, dg in _DG_CACHE:
        if gg is g and dg.device == dev:
            return dg
    dg = DeviceGrammar(g, dev)
    _DG_CACHE.insert(0, (g, dg))
    del _DG_CACHE[2:]
    return dg


def _chart_from_workspace(ws: torch.Tensor, shape, n_nt: int, length: int,
                          unary_row: np.ndarray, meter: AllocMeter | None = None) -> InsideChart:
    """Copy one sentence's chart (batch row 0) to the reference layout.

    The engine stores base-2 offsets from an fp64 per-span shift x; the
    natural-log chart value is ln2 * (x[row] + offset[row, A])."""
    lay = _lib.chart_layout(shape)
    np_, l = int(lay.np), shape.max_len
    B = shape.batch
    n_sym = n_nt + unary_row.shape[1]
    ln2 = math.log(2.0)
    xs = ws[int(lay.off_x):int(lay.off_x) + 8 * int(lay.rows)].view(torch.float64).cpu().numpy()

    meter = meter or AllocMeter()

    def full(shape_):  # the exported chart arrays are retained (inside.py:52-60)
        a = meter.alloc(shape_, retained=True)
        a.fill(NEG_INF)
        return a

    def rows(off, w, half=False):
        base = B * ((w - 1) * (l + 1) - (w - 1) * w // 2)
        n = length - w + 1
        esz = 2 if half else 4
        start = off + esz * base * np_
        flat = ws[start:start + esz * n * np_].view(torch.float16 if half else torch.float32)
        rel = flat.view(n, np_)[:, :n_nt].double().cpu().numpy()
        if half:  # fp16 linear acc * 2^14 (flashinside.h, FI_CHART_F16)
            with np.errstate(divide="ignore"):
                rel = np.log2(rel) - 14.0
        return ln2 * (xs[base:base + n, None] + rel)

    half_ab = int(lay.chart_fmt) == _lib.FI_CHART_F16

    o = [None] * (length + 1)
    a = [None] * length
    b = [None] * length
    o1 = full((length, n_sym))
    o1[:, n_nt:] = unary_row[:length]          # exact float64 copy (inside.py:390)
    o[1] = o1
    for w in range(1, length + 1):
        if w >= 2:
            ow = full((length - w + 1, n_sym))
            ow[:, :n_nt] = rows(int(lay.off_o), w)
            o[w] = ow
        if w < length:
            a[w] = full((length - w + 1, n_nt))
            a[w][:] = rows(int(lay.off_a), w, half_ab)
            b[w] = full((length - w + 1, n_nt))
            b[w][:] = rows(int(lay.off_b), w, half_ab)
    return InsideChart(length, o, a, b, NEG_INF)


def inside_b200(g, tokens, meter: AllocMeter | None = None,
                gemm_dtype: str = DEFAULT_GEMM_DTYPE) -> InsideChart:
    """ENGINES entry: inside chart of one sentence on the B200 engine.

    Same contract as inside_flash (inside.py:274-340): validates tokens,
    returns an InsideChart whose o[1] is the exact float64 emission gather,
    and keeps the device state so inside_backward_b200 can recompute."""
    toks = _prepare(g, tokens)
    l = int(toks.size)
    dg = device_grammar(g)
    tok_d = torch.as_tensor(toks, device=dg.device).view(1, l)
    unary = dg.unary(tok_d)
    lengths = torch.tensor([l], dtype=torch.int32, device=dg.device)
    log_z, ws = inside_fwd(dg.L, dg.R, dg.root, unary, lengths, gemm_dtype, True)
    n_nt = g.dims.n_nt
    shape = _lib.shape(n_nt, g.dims.n_pt, 1, l, gemm_dtype, True)
    unary_row = np.asarray(g.log_emit)[:, toks].T
    chart = _chart_from_workspace(ws, shape, n_nt, l, unary_row, meter)
    chart.log_z = float(log_z.item())
    chart._device = dict(dg=dg, unary=unary, lengths=lengths, log_z=log_z, ws=ws,
                         shape=shape, gemm_dtype=gemm_dtype, tokens=toks)
    if meter is not None:
        meter.device(ws.numel())
    return chart


def inside_backward_b200(g, tokens, chart: InsideChart):
    """Gradients and span marginals of one sentence (inside.py:375-430).

    Raises InsideError on the reference's conditions: chart/sentence
    mismatch (:387-391) and zero-probability sentences (:392-393)."""
    toks = _prepare(g, tokens)
    l = int(toks.size)
    if chart.length != l:
        raise InsideError(f"chart length {chart.length} != sentence length {l}")
    st = chart._device
    mismatch = (st is None or not np.array_equal(st["tokens"], toks)
                or not np.array_equal(chart.o[1][:, g.dims.n_nt:],
                                      np.asarray(g.log_emit)[:, toks].T))   # inside.py:390
    if not mismatch and st["dg"].g is not g:
        # the device state holds the forward's grammar: gradients are only
        # meaningful for that same grammar
        og = st["dg"].g
        mismatch = not all(np.array_equal(np.asarray(getattr(og, k)), np.asarray(getattr(g, k)))
                           for k in ("log_root", "log_left", "log_right", "log_emit"))
    if mismatch:
        raise InsideError("chart was not produced from this grammar and sentence")
    if not np.isfinite(chart.log_z):
        raise InsideError("zero-probability sentence; gradients undefined")
    dg = st["dg"]
    grad_out = torch.ones(1, dtype=torch.float32, device=dg.device)
    dL, dR, droot, dunary = inside_bwd(grad_out, dg.L, dg.R, dg.root, st["unary"],
                                       st["lengths"], st["log_z"], st["ws"],
                                       st["gemm_dtype"], True)
    n_nt, n_pt, V = g.dims.n_nt, g.dims.n_pt, g.dims.vocab_size
    grad = GrammarGrad.zeros(g.dims)
    grad.d_left[:] = dL.double().cpu().numpy()
    grad.d_right[:] = dR.double().cpu().numpy()
    grad.d_root[:] = droot.double().cpu().numpy()
    du = dunary[0].double().cpu().numpy()                  # (l, P) = go[1][:, N:]
    acc = np.zeros((V, n_pt))
    np.add.at(acc, toks, du)                               # inside.py:420-423
    grad.d_emit[:] = acc.T
    # marginals mu_sym[w] = go[w][:, :N]  (inside.py:425-430)
    shape = st["shape"]
    lay = _lib.chart_layout(shape)
    first = shape.batch * l                                 # rowbase(2) = B * l
    total = int(lay.rows) - first
    mu_flat = torch.empty(total, n_nt, dtype=torch.float32, device=dg.device)
    lib = _lib.load()
    _lib.check(lib.fi_marginals(ctypes.byref(shape), _p(st["lengths"]), _p(grad_out),
                                _p(mu_flat), _p(st["ws"]), _stream(dg.device)))
    mu_np = mu_flat.double().cpu().numpy()
    mu_sym = [None, None]
    mu = [None, None]
    pos = 0
    for w in range(2, l + 1):
        n = l - w + 1
        mu_sym.append(mu_np[pos:pos + n].copy())
        mu.append(mu_sym[-1].sum(axis=1))
        pos += n
    return grad, MarginalTable(l, mu, mu_sym)


ENGINES = {"b200": inside_b200}


def register(registry: dict, name: str = "b200") -> dict:
    """Install the engine into a reference-style registry (inside.py:343-348)."""
    registry[name] = inside_b200
    return registry


def batched_inside(g, sentences, gemm_dtype: str = DEFAULT_GEMM_DTYPE,
                   dg: DeviceGrammar | None = None) -> np.ndarray:
    """log_z of every sentence, in equal-length device batches."""
    sents = [_prepare(g, s) for s in sentences]
    dg = dg or device_grammar(g)
    out = np.empty(len(sents))
    by_len: dict[int, list[int]] = {}
    for k, s in enumerate(sents):
        by_len.setdefault(int(s.size), []).append(k)
    with torch.no_grad():
        for l, idx in sorted(by_len.items()):
            toks = torch.as_tensor(np.stack([sents[k] for k in idx]), device=dg.device)
            lengths = torch.full((len(idx),), l, dtype=torch.int32, device=dg.device)
            log_z, _ = inside_fwd(dg.L, dg.R, dg.root, dg.unary(toks), lengths, gemm_dtype,
                                  False)
            out[idx] = log_z.double().cpu().numpy()
    return out


def corpus_log_likelihood(g, sentences, engine: str = "b200",
                          gemm_dtype: str = DEFAULT_GEMM_DTYPE):
    """Per-sentence log-likelihoods and per-token perplexity (inside.py:555-578)."""
    if engine not in ENGINES:
        raise InsideError(f"unknown engine {engine!r}; choose from {sorted(ENGINES)}")
    sentences = list(sentences)
    if not sentences:
        raise InsideError("empty corpus")
    for idx, sent in enumerate(sentences):
        try:
            _prepare(g, sent)
        except InsideError as e:
            raise InsideError(f"sentence {idx}: {e}") from e
    log_likes = batched_inside(g, sentences, gemm_dtype)
    n_tokens = sum(len(s) for s in sentences)
    ppl = float(np.exp(-np.sum(log_likes) / n_tokens))
    return [float(v) for v in log_likes], ppl
