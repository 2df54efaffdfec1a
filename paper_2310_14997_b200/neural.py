"""Grammar parameterisations and the batched training step on the GPU
(the producer of the op's L, R, root, unary).

Mirrors /root/reference/pkg/src/flashpcfg/neuralparam.py and the per-batch
step of train.py, with the same names and semantics:

* ``init_params``        neuralparam.py:86-102  same RNG draw order as the
                         reference (Xavier-normal weights, scaled-normal
                         embeddings, zero biases): identical tensors per seed
* ``grammar_tables``     neuralparam.py:149-208 (``_Forward``): root from
                         f1(start) . u_nt, left/right from f3(parent) .
                         f2/f4(child), emission from f5(preterminal) . u_voc,
                         each row log-softmaxed; ``tied`` reuses the left head
* backward               neuralparam.py:242-320 (``backward_params``) is torch
                         autograd through the same graph; gradients are checked
                         against the reference's manual backward in the tests
* ``init_direct`` / direct tables  neuralparam.py:359-389
* ``clip_grads_``        train.py:133-142 (global norm)
* ``adam_step``          neuralparam.py:337-354 (bias-corrected Adam)
* ``TrainStep``          train.py:201-227: tables -> unary gather -> inside op
                         (fwd+bwd on the sm_100a engine) -> loss = -mean log Z
                         -> backward -> (data-parallel all-reduce of the
                         PARAMETER gradients) -> clip -> Adam

The four score tables (N x d by d x (N+P) products + row log-softmax, and
their backward) run on this repo's engine (``score_table``:
fi_param_scores / fi_param_scores_backward, the tcgen05 GEMM); the residual
MLP layers (d x d) are plain library GEMMs; the inside algorithm runs on the
engine.  With data parallelism the single collective is an
all-reduce of the parameter gradients (~9.2 M + 512 V floats at N = 4096,
d = 512), not of dL and dR (67 M floats).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.distributed as dist
import torch.nn.functional as F

from . import _lib
from .dp import allreduce_grads
from .grammar import GrammarDims
from .ops import _p, _stream, inside


class ParamError(Exception):
    """Invalid parameters or a non-finite value (neuralparam.py:24-25)."""


class TrainError(Exception):
    """A diverged training run: non-finite loss (train.py:33-34, :209-212)."""


def tensor_shapes(dims: GrammarDims, d: int) -> dict[str, tuple[int, ...]]:
    """Names and shapes of the embedding parameterisation (neuralparam.py:70-83)."""
    shapes: dict[str, tuple[int, ...]] = {
        "w_sym": (1 + dims.n_nt + dims.n_pt, d),  # start symbol, nonterminals, preterminals
        "u_nt": (dims.n_nt, d),
        "u_voc": (dims.vocab_size, d),
    }
    for blk in ("f1", "f5"):  # two residual two-layer blocks each
        for k in range(1, 5):
            shapes[f"{blk}.w{k}"] = (d, d)
        for k in range(1, 5):
            shapes[f"{blk}.b{k}"] = (d,)
    for blk in ("f2", "f3", "f4"):  # single relu layer with a residual connection
        shapes[f"{blk}.w"] = (d, d)
        shapes[f"{blk}.b"] = (d,)
    return shapes


@dataclass
class EmbeddingParams:
    """Named parameter tensors (neuralparam.py:42-67), here torch tensors."""

    dims: GrammarDims
    d: int
    tensors: dict[str, torch.Tensor]


def init_params(dims: GrammarDims, d: int = 512, seed: int = 0, device=None,
                dtype=torch.float32) -> EmbeddingParams:
    """Fresh parameters drawn exactly as the reference's init_params."""
    if d < 2:
        raise ParamError(f"embedding dimension must be at least 2, got {d}")
    rng = np.random.default_rng(seed)
    out: dict[str, torch.Tensor] = {}
    for name, shape in tensor_shapes(dims, d).items():
        if name in ("w_sym", "u_nt", "u_voc"):
            a = rng.standard_normal(shape) / math.sqrt(d)
        elif len(shape) == 2:
            n_out, n_in = shape
            a = rng.normal(0.0, math.sqrt(2.0 / (n_in + n_out)), size=shape)
        else:
            a = np.zeros(shape)
        out[name] = torch.tensor(a, dtype=dtype, device=device)
    return EmbeddingParams(dims, d, out)


def _residual_relu(x, w, b):
    return torch.relu(x @ w.T + b) + x


def _two_layer(x, w1, b1, w2, b2):
    return x + torch.relu(x @ w1.T + b1) @ w2.T + b2


class _ScoreTable(torch.autograd.Function):
    """log_softmax(A B^T, rows) on the engine (fi_param_scores /
    fi_param_scores_backward: the tcgen05 GEMM + row log-softmax passes)."""

    @staticmethod
    def forward(ctx, A, B, gemm_dtype):
        A = A.contiguous()
        B = B.contiguous()
        rows, d = A.shape
        cols = B.shape[0]
        mode = _lib.GEMM_DTYPES[gemm_dtype]
        lib = _lib.load()
        ws = torch.empty(lib.fi_param_workspace_bytes(mode, rows, cols, d), dtype=torch.uint8,
                         device=A.device)
        logp = torch.empty(rows, cols, dtype=torch.float32, device=A.device)
        with torch.cuda.device(A.device):
            _lib.check(lib.fi_param_scores(mode, rows, cols, d, _p(A), _p(B), _p(logp), _p(ws),
                                           _stream(A.device)))
        ctx.save_for_backward(A, B, logp)
        ctx.mode = mode
        return logp

    @staticmethod
    def backward(ctx, dlogp):
        A, B, logp = ctx.saved_tensors
        rows, d = A.shape
        cols = B.shape[0]
        lib = _lib.load()
        dlogp = dlogp.contiguous().to(torch.float32)
        ws = torch.empty(lib.fi_param_workspace_bytes(ctx.mode, rows, cols, d),
                         dtype=torch.uint8, device=A.device)
        dA = torch.empty_like(A)
        dB = torch.empty_like(B)
        with torch.cuda.device(A.device):
            _lib.check(lib.fi_param_scores_backward(ctx.mode, rows, cols, d, _p(A), _p(B),
                                                    _p(logp), _p(dlogp), _p(dA), _p(dB), _p(ws),
                                                    _stream(A.device)))
        return dA, dB, None


def score_table(A: torch.Tensor, B: torch.Tensor, gemm_dtype: str = "fp32") -> torch.Tensor:
    """log_softmax(A @ B.T, dim=-1) of fp32 CUDA tensors on the engine's kernels
    (neuralparam.py:185-189); differentiable in A and B.  tf32 products for
    gemm_dtype "bf16" / "tf32", bf16x3 split products for "fp32" (parity)."""
    if not (A.is_cuda and B.is_cuda) or A.dtype != torch.float32 or B.dtype != torch.float32:
        raise ValueError("score_table needs fp32 CUDA tensors (the engine has no CPU path)")
    return _ScoreTable.apply(A, B, gemm_dtype)


def grammar_tables(p: EmbeddingParams, tied: bool = False, finite_flags: list | None = None,
                   gemm_dtype: str = "fp32"):
    """(log_root (N,), log_left (N, N+P), log_right, log_emit (P, V)), differentiable,
    on the GPU: the residual MLPs (d x d layers, library GEMMs) and the four
    score tables on the engine (``score_table``).  Same graph as
    ``grammar_tables_torch``, the plain-torch restatement the CPU tests pin
    against the reference (neuralparam.py:149-208)."""
    return _tables(p, tied, finite_flags, lambda a, b: score_table(a, b, gemm_dtype))


def grammar_tables_torch(p: EmbeddingParams, tied: bool = False,
                         finite_flags: list | None = None):
    """The parameterisation in plain torch (any device / dtype, float64 on the
    CPU in tests): the restatement of neuralparam.py:149-208 that
    ``grammar_tables`` runs on the engine.

    Non-finite activations raise ParamError (neuralparam.py); with
    ``finite_flags`` the per-activation checks are appended there as device
    booleans instead (no host sync: the caller checks them once)."""
    return _tables(p, tied, finite_flags, lambda a, b: F.log_softmax(a @ b.T, dim=-1))


def _tables(p: EmbeddingParams, tied: bool, finite_flags: list | None, scores):

    def check(name, a):
        if finite_flags is not None:
            finite_flags.append((name, torch.isfinite(a).all()))
        elif not torch.isfinite(a).all():
            raise ParamError(f"non-finite activation in {name}")

    t = p.tensors
    n = p.dims.n_nt
    x_start = t["w_sym"][0:1]
    x_nt = t["w_sym"][1:1 + n]
    x_child = t["w_sym"][1:]
    x_pt = t["w_sym"][1 + n:]
    f1 = _two_layer(_two_layer(x_start, t["f1.w1"], t["f1.b1"], t["f1.w2"], t["f1.b2"]),
                    t["f1.w3"], t["f1.b3"], t["f1.w4"], t["f1.b4"])
    f3 = _residual_relu(x_nt, t["f3.w"], t["f3.b"])
    f2 = _residual_relu(x_child, t["f2.w"], t["f2.b"])
    f5 = _two_layer(_two_layer(x_pt, t["f5.w1"], t["f5.b1"], t["f5.w2"], t["f5.b2"]),
                    t["f5.w3"], t["f5.b3"], t["f5.w4"], t["f5.b4"])
    for name, a in (("f1", f1), ("f2", f2), ("f3", f3), ("f5", f5)):
        check(name, a)
    log_root = scores(f1, t["u_nt"])[0]
    log_left = scores(f3, f2)
    if tied:
        log_right = log_left
    else:
        f4 = _residual_relu(x_child, t["f4.w"], t["f4.b"])
        check("f4", f4)
        log_right = scores(f3, f4)
    log_emit = scores(f5, t["u_voc"])
    return log_root, log_left, log_right, log_emit


@dataclass
class DirectLogits:
    """Raw score tables softmaxed row-wise (neuralparam.py:359-375)."""

    dims: GrammarDims
    tensors: dict[str, torch.Tensor]


def init_direct(dims: GrammarDims, seed: int = 0, scale: float = 0.5, device=None,
                dtype=torch.float32) -> DirectLogits:
    rng = np.random.default_rng(seed)
    shapes = (("root", (dims.n_nt,)), ("left", (dims.n_nt, dims.n_sym)),
              ("right", (dims.n_nt, dims.n_sym)), ("emit", (dims.n_pt, dims.vocab_size)))
    return DirectLogits(dims, {k: torch.tensor(scale * rng.standard_normal(s), dtype=dtype,
                                               device=device) for k, s in shapes})


def direct_tables(p: DirectLogits, tied: bool = False):
    """Row log-softmax of the raw tables (neuralparam.py:359-375); elementwise
    library ops (no product to put on the engine)."""
    t = p.tensors
    log_left = F.log_softmax(t["left"], dim=-1)
    log_right = log_left if tied else F.log_softmax(t["right"], dim=-1)
    return (F.log_softmax(t["root"], dim=-1), log_left, log_right,
            F.log_softmax(t["emit"], dim=-1))


# --------------------------------------------------------------- optimiser
@dataclass
class AdamState:
    """First / second moments and the step counter (neuralparam.py:325-334)."""

    m: dict[str, torch.Tensor]
    v: dict[str, torch.Tensor]
    t: int = 0

    @staticmethod
    def zeros(tensors: dict[str, torch.Tensor]) -> "AdamState":
        return AdamState({k: torch.zeros_like(x) for k, x in tensors.items()},
                         {k: torch.zeros_like(x) for k, x in tensors.items()})


def grad_norm(grads: dict[str, torch.Tensor]) -> torch.Tensor:
    """Joint L2 norm of all gradients (a device scalar: no host sync)."""
    return torch.linalg.vector_norm(torch.stack([torch.linalg.vector_norm(x)
                                                 for x in grads.values()]))


def clip_grads_(grads: dict[str, torch.Tensor], max_norm: float) -> torch.Tensor:
    """Scale all gradients so their joint norm is at most max_norm (train.py:133-142).
    Returns the pre-clip norm (a device scalar: no host sync)."""
    norm = grad_norm(grads)
    torch._foreach_mul_(list(grads.values()), torch.clamp(max_norm / norm, max=1.0))
    return norm


def adam_step(tensors: dict[str, torch.Tensor], grads: dict[str, torch.Tensor],
              state: AdamState, lr: float = 0.002, beta1: float = 0.75,
              beta2: float = 0.999, eps: float = 1e-8, check_finite: bool = True) -> None:
    """One bias-corrected Adam update in place (neuralparam.py:337-354):
    x -= lr * (m / (1 - b1^t)) / (sqrt(v / (1 - b2^t)) + eps)."""
    names = list(tensors)
    if check_finite:
        bad = [k for k in names if not torch.isfinite(grads[k]).all()]
        if bad:
            raise ParamError(f"non-finite gradient for {bad[0]}")
    state.t += 1
    c1 = 1.0 - beta1 ** state.t
    c2 = 1.0 - beta2 ** state.t
    xs = [tensors[k] for k in names]
    gs = [grads[k] for k in names]
    ms = [state.m[k] for k in names]
    vs = [state.v[k] for k in names]
    torch._foreach_mul_(ms, beta1)
    torch._foreach_add_(ms, gs, alpha=1.0 - beta1)
    torch._foreach_mul_(vs, beta2)
    torch._foreach_addcmul_(vs, gs, gs, value=1.0 - beta2)
    denom = torch._foreach_div(vs, c2)
    torch._foreach_sqrt_(denom)
    torch._foreach_add_(denom, eps)
    step = torch._foreach_div(ms, denom)
    torch._foreach_add_(xs, step, alpha=-lr / c1)


# ------------------------------------------------------------ training step
@dataclass
class TrainConfig:
    """The optimiser / model knobs of the reference TrainConfig (train.py:38-57)."""

    parameterization: str = "neural"
    d: int = 512
    lr: float = 0.002
    beta1: float = 0.75
    beta2: float = 0.999
    eps: float = 1e-8
    clip: float = 5.0
    tied: bool = False
    gemm_dtype: str = "bf16"


@dataclass
class TrainStep:
    """One optimisation step of train.py:201-227 on the GPU, batched.

    ``step(tokens, lengths)`` takes a (B, lmax) int64 token tensor and
    (B,) int32 lengths on the device; returns the mean per-sentence NLL
    (a device scalar).  Under torch.distributed each rank passes its shard
    of the batch; the parameter gradients are summed with ONE all-reduce
    of a flat buffer and the loss is the global mean (every rank applies
    the identical update)."""

    params: EmbeddingParams | DirectLogits
    config: TrainConfig = field(default_factory=TrainConfig)
    state: AdamState | None = None

    def __post_init__(self):
        for x in self.params.tensors.values():
            x.requires_grad_(True)
        if self.state is None:
            self.state = AdamState.zeros({k: v.detach() for k, v in self.params.tensors.items()})

    def tables(self, finite_flags: list | None = None):
        if isinstance(self.params, EmbeddingParams):
            return grammar_tables(self.params, self.config.tied, finite_flags,
                                  self.config.gemm_dtype)
        return direct_tables(self.params, self.config.tied)

    def _forward_backward(self, tokens: torch.Tensor, lengths: torch.Tensor, denom: float):
        """tables -> unary gather -> inside fwd+bwd on the engine -> autograd
        through the tables (the train.py:208-224 chain, batched) with
        loss = -sum(log Z) / denom.  Returns (loss, grads, log_z, checks):
        ``checks`` are device booleans queued with the step and read once by
        the caller (no host sync in front of the engine)."""
        cfg = self.config
        xs = list(self.params.tensors.values())
        flags: list = []
        # the score-table GEMMs (N x d x (N+P)) run on TF32 tensor cores in the
        # fast modes; fp32 mode keeps exact fp32 products (parity mode)
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = cfg.gemm_dtype != "fp32"
        try:
            log_root, log_left, log_right, log_emit = self.tables(flags)
            # inside.py:296-298 as a row lookup in the (V, P) transpose: coalesced
            # rows and the embedding backward (fwd+bwd 156 -> 101 us at config 3)
            unary = F.embedding(tokens, log_emit.T.contiguous())
            # lengths are checked with the other deferred flags (validate=False:
            # an invalid one makes its sentence inert with log Z = NaN)
            flags.append(("lengths", ((lengths >= 2) & (lengths <= tokens.shape[1])).all()))
            log_z = inside(log_left.contiguous(), log_right.contiguous(), log_root.contiguous(),
                           unary.contiguous(), lengths, gemm_dtype=cfg.gemm_dtype,
                           validate=False)
            loss = -log_z.sum() / denom                                # train.py:218: -1/B
            grads = torch.autograd.grad(loss, xs, allow_unused=True)  # tied: f4 unused
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev
        grads = [torch.zeros_like(x) if g is None else g for x, g in zip(xs, grads)]
        return loss, grads, log_z, flags

    def _raise_on(self, flags, ok, log_z, lengths, loss_finite: bool, grad_finite: bool,
                  step_no: int):
        """The reference's error order: a non-finite activation (ParamError,
        raised while the grammar is built), an invalid sentence length
        (inside.py:113-121), a non-finite log Z (TrainError, train.py:209-212),
        a non-finite gradient (ParamError, neuralparam.py:341-343) -- all
        before any parameter is touched."""
        for (name, _), good in zip(flags, ok):
            if not good:
                if name == "lengths":
                    b = int(((lengths < 2) | (lengths > self._lmax)).nonzero()[0, 0])
                    raise ValueError(f"sentence {b}: length {int(lengths[b])} outside "
                                     f"[2, {self._lmax}]")
                raise ParamError(f"non-finite activation in {name}")
        if not loss_finite:
            bad = (~torch.isfinite(log_z)).nonzero()
            if bad.numel():  # this rank holds the sentence (else another rank does)
                b = int(bad[0, 0])
                raise TrainError(f"non-finite loss at step {step_no}: sentence {b} has log "
                                 f"probability {float(log_z[b].detach())}")
            raise TrainError(f"non-finite loss at step {step_no} (on another rank)")
        if not grad_finite:
            raise ParamError("non-finite gradient")

    def loss_and_grads(self, tokens: torch.Tensor, lengths: torch.Tensor,
                       global_batch: int | None = None):
        """Loss = -sum(log Z) / global_batch and its parameter gradients on this
        rank (no collective); raises like the reference before returning."""
        self._lmax = int(tokens.shape[1])
        loss, grads, log_z, flags = self._forward_backward(tokens, lengths,
                                                           float(global_batch or tokens.shape[0]))
        ok = torch.stack([f for _, f in flags] + [torch.isfinite(loss)]).cpu().tolist()
        self._raise_on(flags, ok[:-1], log_z, lengths, ok[-1], True, self.state.t + 1)
        return loss, grads

    def step(self, tokens: torch.Tensor, lengths: torch.Tensor, global_batch: int | None = None,
             group=None) -> torch.Tensor:
        """One optimisation step; returns the global mean NLL (device scalar).

        Under torch.distributed the parameter gradients, the loss and (when
        ``global_batch`` is not given) the sentence count travel in ONE flat
        all-reduce, so uneven shards still average over the global batch."""
        cfg = self.config
        names = list(self.params.tensors)
        xs = [self.params.tensors[k] for k in names]
        self._lmax = int(tokens.shape[1])
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        count_in_bucket = world > 1 and global_batch is None
        denom = 1.0 if count_in_bucket else float(global_batch or tokens.shape[0])
        loss, grads, log_z, flags = self._forward_backward(tokens, lengths, denom)
        if world > 1:  # one collective: [parameter grads | loss | sentence count]
            extra = [loss.detach().reshape(1)]
            if count_in_bucket:
                extra.append(torch.full((1,), float(tokens.shape[0]), device=loss.device))
            out = allreduce_grads(list(grads) + extra, group)
            grads, loss = out[:len(grads)], out[len(grads)][0]
            if count_in_bucket:  # the global mean over however the batch was sharded
                count = out[-1][0]
                grads = [g / count for g in grads]
                loss = loss / count
        gd = dict(zip(names, grads))
        norm = grad_norm(gd)
        ok = torch.stack([f for _, f in flags] + [torch.isfinite(loss), torch.isfinite(norm)])
        ok = ok.cpu().tolist()  # the step's single host read
        self._raise_on(flags, ok[:-2], log_z, lengths, ok[-2], ok[-1], self.state.t + 1)
        torch._foreach_mul_(list(gd.values()), torch.clamp(cfg.clip / norm, max=1.0))
        with torch.no_grad():
            adam_step({k: x.data for k, x in zip(names, xs)}, gd, self.state, lr=cfg.lr,
                      beta1=cfg.beta1, beta2=cfg.beta2, eps=cfg.eps, check_finite=False)
        return loss.detach()
