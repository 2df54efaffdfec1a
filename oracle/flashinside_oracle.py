"""CPU oracle for the FlashInside hot path -- TEST INFRASTRUCTURE ONLY.

A float64 NumPy restatement of the reference's inside algorithm
(/root/reference/pkg/src/flashpcfg/inside.py), used only as the checker by
tests/, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` leg of bench.py.
The product path (paper_2310_14997_b200) never imports it.

Parity is pinned: tests/test_oracle.py checks this module against golden
vectors produced by the reference itself (tests/golden/make_golden.py, run
where /root/reference exists): closed-form G1 values, brute-force instances,
chart-level o/a/b, the 512-symbol agreement case, log_z at the SURVEY
configs, and full GrammarGrad / dunary at small sizes.

Restatement notes
* forward  = ``inside_flash`` (inside.py:274-340): width-1 row from the
  emission gather (:296-298), stacked projection with a scalar per-span
  shift (:203-213), split merge by log-sum-exp over split points
  (:313-332), root log-sum-exp (:124-129).  The -inf blocks of the chart
  (NT slots at width 1, PT slots above) contribute exact zeros to the
  projection, so the products are restricted to the live block.
* backward = ``inside_backward`` + ``_projection_backward``
  (inside.py:375-447) in GEMM form: the child softmax
  exp(L + o - a) * ga summed over spans is  W * (G^T E)  and summed over
  parents is  E * (G W)  with  E = exp(o - x), G = ga * exp(x - a)
  (0 where a = -inf, the NaN guard of :441-443).  Mathematically identical
  to the reference's (n, N, n_sym) broadcast; tests gate it against the
  reference's own gradients.
"""

from __future__ import annotations

import numpy as np

NEG_INF = float("-inf")


def _safe_max(x: np.ndarray) -> np.ndarray:
    m = x.max(axis=-1)
    return np.where(np.isfinite(m), m, 0.0)


def _lse(x: np.ndarray, axis: int) -> np.ndarray:
    m = x.max(axis=axis)
    safe = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        return safe + np.log(np.exp(x - np.expand_dims(safe, axis)).sum(axis=axis))


def _project(o_live: np.ndarray, w_live: np.ndarray, n_nt: int):
    """[a | b] = x + log(exp(o - x) @ W^T) over the live block (inside.py:203-213)."""
    x = _safe_max(o_live)
    e = np.exp(o_live - x[:, None])
    with np.errstate(divide="ignore"):
        proj = np.log(e @ w_live.T) + x[:, None]
    return proj[:, :n_nt], proj[:, n_nt:], x, e


class SentenceChart:
    """Per-width chart of one sentence in the reference layout (inside.py:66-84),
    plus the shifts and shifted exponentials the backward reuses."""

    def __init__(self, length: int):
        self.length = length
        self.o = [None] * (length + 1)   # o[w]: (n_w, n_sym)
        self.a = [None] * length         # a[w]: (n_w, N)
        self.b = [None] * length
        self.x = [None] * length
        self.e = [None] * length         # exp(o[w] - x) over the live block
        self.log_z = NEG_INF


def inside_sentence(L, R, root, unary_row) -> SentenceChart:
    """Forward chart of one sentence.  unary_row: (l, P) = log_emit[:, toks].T."""
    n_nt = L.shape[0]
    n_sym = L.shape[1]
    l = unary_row.shape[0]
    w_nn = np.exp(np.concatenate([L[:, :n_nt], R[:, :n_nt]], axis=0))    # (2N, N)
    w_np = np.exp(np.concatenate([L[:, n_nt:], R[:, n_nt:]], axis=0))    # (2N, P)
    ch = SentenceChart(l)
    o1 = np.full((l, n_sym), NEG_INF)
    o1[:, n_nt:] = unary_row
    ch.o[1] = o1
    for w in range(1, l + 1):
        n = l - w + 1
        if w >= 2:
            # split m of span (i, i+w): a[m][i] + b[w-m][i+m]   (inside.py:317-319)
            t = np.stack([ch.a[m][:n] + ch.b[w - m][m:m + n] for m in range(1, w)])
            ow = np.full((n, n_sym), NEG_INF)
            ow[:, :n_nt] = _lse(t, 0)
            ch.o[w] = ow
        if w < l:
            if w == 1:
                a, b, x, e = _project(ch.o[1][:, n_nt:], w_np, n_nt)
            else:
                a, b, x, e = _project(ch.o[w][:, :n_nt], w_nn, n_nt)
            ch.a[w], ch.b[w], ch.x[w], ch.e[w] = a, b, x, e
    scores = root + ch.o[l][0, :n_nt]                                     # inside.py:124-129
    m = scores.max()
    ch.log_z = float(m + np.log(np.exp(scores - m).sum())) if np.isfinite(m) else NEG_INF
    return ch


def backward_sentence(L, R, root, ch: SentenceChart, grad: float = 1.0):
    """GEMM-form inside_backward (inside.py:375-447) of one sentence.

    Returns (dW_nn (2N, N) unscaled-by-W accumulator, dW_np (2N, P),
    d_root (N,), d_unary (l, P), go list) all multiplied by ``grad``."""
    n_nt = L.shape[0]
    n_sym = L.shape[1]
    n_pt = n_sym - n_nt
    l = ch.length
    w_nn = np.exp(np.concatenate([L[:, :n_nt], R[:, :n_nt]], axis=0))
    w_np = np.exp(np.concatenate([L[:, n_nt:], R[:, n_nt:]], axis=0))
    go = [None] + [np.zeros((l - w + 1, n_sym)) for w in range(1, l + 1)]
    ga = [None] + [np.zeros((l - w + 1, n_nt)) for w in range(1, l)]
    gb = [None] + [np.zeros((l - w + 1, n_nt)) for w in range(1, l)]
    acc_nn = np.zeros((2 * n_nt, n_nt))
    acc_np = np.zeros((2 * n_nt, n_pt))
    post = np.exp(root + ch.o[l][0, :n_nt] - ch.log_z)                   # inside.py:402-404
    go[l][0, :n_nt] = post
    d_root = post.copy()
    for w in range(l, 1, -1):
        n = l - w + 1
        gout = go[w][:, :n_nt]
        o_w = ch.o[w][:, :n_nt]
        for m in range(1, w):                                            # inside.py:410-417
            with np.errstate(invalid="ignore"):
                t = ch.a[m][:n] + ch.b[w - m][m:m + n] - o_w
            t[np.isnan(t)] = NEG_INF
            t = np.exp(t) * gout
            ga[m][:n] += t
            gb[w - m][m:m + n] += t
        m = w - 1                                                        # inside.py:433-447
        with np.errstate(over="ignore", invalid="ignore"):
            gl = np.where(np.isneginf(ch.a[m]), 0.0, ga[m] * np.exp(ch.x[m][:, None] - ch.a[m]))
            gr = np.where(np.isneginf(ch.b[m]), 0.0, gb[m] * np.exp(ch.x[m][:, None] - ch.b[m]))
        g = np.concatenate([gl, gr], axis=1)                             # (n_m, 2N)
        if m >= 2:
            go[m][:, :n_nt] += ch.e[m] * (g @ w_nn)
            acc_nn += g.T @ ch.e[m]
        else:
            go[1][:, n_nt:] += ch.e[1] * (g @ w_np)
            acc_np += g.T @ ch.e[1]
    d_unary = go[1][:, n_nt:].copy()
    return (grad * acc_nn, grad * acc_np, grad * d_root, grad * d_unary, go)


def inside_batch(L, R, root, unary, lengths, grad_log_z=None, backward=True):
    """Batched oracle matching the engine's op contract.

    unary (B, lmax, P); lengths (B,).  Returns dict with log_z (B,) and, if
    backward, dL, dR (N, N+P), droot (N,), dunary (B, lmax, P)."""
    L = np.asarray(L, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    root = np.asarray(root, dtype=np.float64)
    unary = np.asarray(unary, dtype=np.float64)
    lengths = np.asarray(lengths, dtype=np.int64)
    n_nt, n_sym = L.shape
    bsz, lmax, n_pt = unary.shape
    if grad_log_z is None:
        grad_log_z = np.ones(bsz)
    out = {"log_z": np.zeros(bsz), "charts": []}
    acc_nn = np.zeros((2 * n_nt, n_nt))
    acc_np = np.zeros((2 * n_nt, n_pt))
    droot = np.zeros(n_nt)
    dunary = np.zeros((bsz, lmax, n_pt))
    for b in range(bsz):
        ch = inside_sentence(L, R, root, unary[b, :lengths[b]])
        out["log_z"][b] = ch.log_z
        out["charts"].append(ch)
        if backward and grad_log_z[b] != 0.0 and np.isfinite(ch.log_z):
            ann, anp, dr, du, _ = backward_sentence(L, R, root, ch, float(grad_log_z[b]))
            acc_nn += ann
            acc_np += anp
            droot += dr
            dunary[b, :lengths[b]] = du
    if backward:
        dL = np.zeros_like(L)
        dR = np.zeros_like(R)
        dL[:, :n_nt] = np.exp(L[:, :n_nt]) * acc_nn[:n_nt]
        dR[:, :n_nt] = np.exp(R[:, :n_nt]) * acc_nn[n_nt:]
        dL[:, n_nt:] = np.exp(L[:, n_nt:]) * acc_np[:n_nt]
        dR[:, n_nt:] = np.exp(R[:, n_nt:]) * acc_np[n_nt:]
        out.update(dL=dL, dR=dR, droot=droot, dunary=dunary)
    return out


def inside_batch_equal(L, R, root, unary, grad_log_z=None, backward=True):
    """``inside_batch`` for a batch of equal-length sentences, vectorised over
    the batch so the BASELINE configs (64 x |N| = 4096, l = 40) check in
    seconds instead of minutes.  Same restatement, line for line, with a
    leading batch axis on every chart array: the projection of width w is
    one (B n_w, K) x (K, 2N) product (inside.py:203-213), the split merge a
    log-sum-exp over m taken in two passes, max then sum (inside.py:323-331),
    the backward the GEMM form of inside.py:375-447 with the upstream
    gradient folded into the root seed (the reference scales each
    sentence's GrammarGrad afterwards: linear, so equal up to rounding).
    Gated against ``inside_batch`` in tests/test_oracle.py."""
    L = np.asarray(L, dtype=np.float64)
    R = np.asarray(R, dtype=np.float64)
    root = np.asarray(root, dtype=np.float64)
    unary = np.asarray(unary, dtype=np.float64)
    n_nt, n_sym = L.shape
    bsz, l, n_pt = unary.shape
    grad = np.ones(bsz) if grad_log_z is None else np.asarray(grad_log_z, dtype=np.float64)
    w_nn = np.exp(np.concatenate([L[:, :n_nt], R[:, :n_nt]], axis=0))    # (2N, N)
    w_np = np.exp(np.concatenate([L[:, n_nt:], R[:, n_nt:]], axis=0))    # (2N, P)
    o = [None] * (l + 1)        # o[w]: (B, n_w, N) NT block (w >= 2); o[1] = unary
    a = [None] * l
    b = [None] * l
    x = [None] * l
    e = [None] * l
    o[1] = unary
    for w in range(1, l + 1):
        n = l - w + 1
        if w >= 2:                                                       # inside.py:313-332
            mx = np.full((bsz, n, n_nt), NEG_INF)
            for m in range(1, w):
                mx = np.maximum(mx, a[m][:, :n] + b[w - m][:, m:m + n])
            sh = np.where(np.isfinite(mx), mx, 0.0)
            acc = np.zeros((bsz, n, n_nt))
            for m in range(1, w):
                acc += np.exp(a[m][:, :n] + b[w - m][:, m:m + n] - sh)
            with np.errstate(divide="ignore"):
                o[w] = sh + np.log(acc)
        if w < l:                                                        # inside.py:203-213
            live = o[w].reshape(bsz * n, -1)
            xs = _safe_max(live)
            ex = np.exp(live - xs[:, None])
            with np.errstate(divide="ignore"):
                proj = np.log(ex @ (w_np if w == 1 else w_nn).T) + xs[:, None]
            a[w] = proj[:, :n_nt].reshape(bsz, n, n_nt)
            b[w] = proj[:, n_nt:].reshape(bsz, n, n_nt)
            x[w] = xs.reshape(bsz, n)
            e[w] = ex.reshape(bsz, n, -1)
    scores = root[None, :] + o[l][:, 0, :]                               # inside.py:124-129
    log_z = _lse(scores, 1)
    out = {"log_z": log_z}
    if not backward:
        return out
    live = np.isfinite(log_z) & (grad != 0.0)
    go = [None] * (l + 1)
    go[1] = np.zeros((bsz, l, n_pt))
    for w in range(2, l + 1):
        go[w] = np.zeros((bsz, l - w + 1, n_nt))
    ga = [None] + [np.zeros((bsz, l - w + 1, n_nt)) for w in range(1, l)]
    gb = [None] + [np.zeros((bsz, l - w + 1, n_nt)) for w in range(1, l)]
    acc_nn = np.zeros((2 * n_nt, n_nt))
    acc_np = np.zeros((2 * n_nt, n_pt))
    with np.errstate(invalid="ignore", over="ignore"):
        post = np.exp(scores - np.where(live, log_z, 0.0)[:, None])      # inside.py:402-404
    post = np.where(live[:, None], post * grad[:, None], 0.0)
    go[l][:, 0, :] = post
    droot = post.sum(axis=0)
    for w in range(l, 1, -1):
        n = l - w + 1
        gout = go[w]
        for m in range(1, w):                                            # inside.py:410-417
            with np.errstate(invalid="ignore"):
                t = a[m][:, :n] + b[w - m][:, m:m + n] - o[w]
            t[np.isnan(t)] = NEG_INF
            t = np.exp(t) * gout
            ga[m][:, :n] += t
            gb[w - m][:, m:m + n] += t
        m = w - 1                                                        # inside.py:433-447
        with np.errstate(over="ignore", invalid="ignore"):
            gl = np.where(np.isneginf(a[m]), 0.0, ga[m] * np.exp(x[m][..., None] - a[m]))
            gr = np.where(np.isneginf(b[m]), 0.0, gb[m] * np.exp(x[m][..., None] - b[m]))
        g = np.concatenate([gl, gr], axis=2).reshape(bsz * (l - m + 1), 2 * n_nt)
        em = e[m].reshape(bsz * (l - m + 1), -1)
        if m >= 2:
            go[m] += (em * (g @ w_nn)).reshape(go[m].shape)
            acc_nn += g.T @ em
        else:
            go[1] += (em * (g @ w_np)).reshape(go[1].shape)
            acc_np += g.T @ em
    dL = np.zeros_like(L)
    dR = np.zeros_like(R)
    dL[:, :n_nt] = np.exp(L[:, :n_nt]) * acc_nn[:n_nt]
    dR[:, :n_nt] = np.exp(R[:, :n_nt]) * acc_nn[n_nt:]
    dL[:, n_nt:] = np.exp(L[:, n_nt:]) * acc_np[:n_nt]
    dR[:, n_nt:] = np.exp(R[:, n_nt:]) * acc_np[n_nt:]
    out.update(dL=dL, dR=dR, droot=droot, dunary=go[1])
    return out


def marginals_sentence(ch: SentenceChart, go) -> list:
    """mu_sym[w] = go[w][:, :N] for w >= 2 (inside.py:425-430)."""
    n_nt = ch.a[1].shape[1]
    return [None, None] + [go[w][:, :n_nt].copy() for w in range(2, ch.length + 1)]


# ---------------------------------------------------------------- fixtures
def random_grammar_arrays(n_nt: int, n_pt: int, vocab: int, seed: int,
                          concentration: float = 1.0):
    """Same draws as grammar.random_grammar (grammar.py:160-180)."""
    rng = np.random.default_rng(seed)

    def rows(r, c):
        p = rng.dirichlet(np.full(c, concentration), size=r)
        with np.errstate(divide="ignore"):
            return np.log(p)

    root = rows(1, n_nt)[0]
    left = rows(n_nt, n_nt + n_pt)
    right = rows(n_nt, n_nt + n_pt)
    emit = rows(n_pt, vocab)
    return root, left, right, emit


def unary_from_tokens(emit: np.ndarray, tokens: np.ndarray, lmax: int | None = None):
    """unary[b, i, T] = emit[T, tokens[b][i]] (inside.py:296-298), zero-padded."""
    seqs = [np.asarray(t, dtype=np.int64) for t in tokens]
    lmax = lmax or max(len(s) for s in seqs)
    out = np.zeros((len(seqs), lmax, emit.shape[0]))
    for b, s in enumerate(seqs):
        out[b, :len(s)] = emit[:, s].T
    return out
