"""PyTorch custom op ``flashinside::inside`` over the C ABI.

    log_z = inside(L, R, root, unary, lengths, gemm_dtype="bf16")

is the batched, differentiable form of the reference's inside pass
(``inside_flash`` + ``inside_backward``, pkg/src/flashpcfg/inside.py:274-447):

* ``L, R``   fp32 (N, N+P)  log_left / log_right  (grammar.py:99-100)
* ``root``   fp32 (N,)      log_root
* ``unary``  fp32 (B, l, P) unary[b, i, T] = log_emit[T, tokens[b][i]]
* ``lengths`` int (B,)      2 <= lengths[b] <= l; padded positions are ignored

Autograd returns dL, dR, droot and dunary (no gradient for lengths).  CUDA
only; there is no CPU path.  PyTorch supplies device memory and the stream;
all compute happens in the sm_100a library.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib


def _p(t: torch.Tensor | None) -> ctypes.c_void_p:
    return ctypes.c_void_p(0 if t is None else t.data_ptr())


def _stream(device: torch.device) -> ctypes.c_void_p:
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _check_inputs(L, R, root, unary, lengths):
    for name, t in (("L", L), ("R", R), ("root", root), ("unary", unary)):
        if not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
        if t.dtype != torch.float32:
            raise ValueError(f"{name} must be float32, got {t.dtype}")
    if lengths.dtype != torch.int32 or not lengths.is_cuda:
        raise ValueError("lengths must be an int32 CUDA tensor")
    if L.dim() != 2 or R.shape != L.shape:
        raise ValueError(f"L and R must have the same (N, N+P) shape, got {tuple(L.shape)} "
                         f"and {tuple(R.shape)}")
    n = root.shape[0]
    if root.dim() != 1 or L.shape[0] != n:
        raise ValueError(f"root must be (N,) with N = L.shape[0]; got {tuple(root.shape)}")
    p = L.shape[1] - n
    if p < 1:
        raise ValueError("L must have at least one preterminal column")
    if unary.dim() != 3 or unary.shape[2] != p:
        raise ValueError(f"unary must be (B, l, P={p}), got {tuple(unary.shape)}")
    if lengths.shape != (unary.shape[0],):
        raise ValueError("lengths must be (B,)")
    return n, p, unary.shape[0], unary.shape[1]


def check_lengths(lengths: torch.Tensor, max_len: int) -> None:
    """Refuse a batch with a sentence outside 2 <= lengths[b] <= max_len before
    any launch (the reference's _prepare, inside.py:113-121, refuses length < 2).

    One device->host read.  Skipped while a CUDA graph is being captured: the
    library's own device-side guard (k_check_lengths) then makes such a
    sentence inert with log Z = NaN and sets FI_FLAG_BAD_LENGTH."""
    if lengths.numel() == 0 or (lengths.is_cuda and torch.cuda.is_current_stream_capturing()):
        return
    bad = (lengths < 2) | (lengths > max_len)
    if bool(bad.any()):
        b = int(bad.nonzero()[0, 0])
        raise ValueError(f"sentence {b}: length {int(lengths[b])} outside [2, {max_len}] "
                         f"(need a token sequence of length >= 2 that fits the padded batch)")


def read_flags(ws: torch.Tensor, shape) -> int:
    """The library's flag word (FI_FLAG_ZERO_PROB | FI_FLAG_BAD_LENGTH) of a workspace."""
    off = int(_lib.chart_layout(shape).off_flag)
    return int(ws[off:off + 4].view(torch.int32).item())


@torch.library.custom_op("flashinside::inside_fwd", mutates_args=())
def inside_fwd(L: torch.Tensor, R: torch.Tensor, root: torch.Tensor, unary: torch.Tensor,
               lengths: torch.Tensor, gemm_dtype: str, store_chart: bool,
               chart_dtype: str = "auto") -> tuple[torch.Tensor, torch.Tensor]:
    L, R, root, unary = (t.contiguous() for t in (L, R, root, unary))
    lengths = lengths.contiguous()
    n, p, b, l = _check_inputs(L, R, root, unary, lengths)
    s = _lib.shape(n, p, b, l, gemm_dtype, store_chart, chart_dtype)
    ws = torch.empty(_lib.workspace_bytes(s), dtype=torch.uint8, device=L.device)
    log_z = torch.empty(b, dtype=torch.float32, device=L.device)
    lib = _lib.load()
    with torch.cuda.device(L.device):
        _lib.check(lib.fi_inside_forward(ctypes.byref(s), _p(L), _p(R), _p(root), _p(unary),
                                         _p(lengths), _p(log_z), _p(ws), _stream(L.device)))
    return log_z, ws


@inside_fwd.register_fake
def _(L, R, root, unary, lengths, gemm_dtype, store_chart, chart_dtype="auto"):
    n, p = root.shape[0], L.shape[1] - root.shape[0]
    s = _lib.shape(n, p, unary.shape[0], unary.shape[1], gemm_dtype, store_chart, chart_dtype)
    return (L.new_empty(unary.shape[0]),
            torch.empty(_lib.workspace_bytes(s), dtype=torch.uint8, device=L.device))


@torch.library.custom_op("flashinside::inside_bwd", mutates_args=("ws",))
def inside_bwd(grad_log_z: torch.Tensor, L: torch.Tensor, R: torch.Tensor, root: torch.Tensor,
               unary: torch.Tensor, lengths: torch.Tensor, log_z: torch.Tensor,
               ws: torch.Tensor, gemm_dtype: str, store_chart: bool, chart_dtype: str = "auto"
               ) -> tuple[torch.Tensor, torch.Tensor, torch.Tensor, torch.Tensor]:
    L, R, root, unary = (t.contiguous() for t in (L, R, root, unary))
    grad_log_z = grad_log_z.contiguous().to(torch.float32)
    n, p, b, l = _check_inputs(L, R, root, unary, lengths)
    s = _lib.shape(n, p, b, l, gemm_dtype, store_chart, chart_dtype)
    dL = torch.empty_like(L)
    dR = torch.empty_like(R)
    droot = torch.empty_like(root)
    dunary = torch.empty_like(unary)
    lib = _lib.load()
    with torch.cuda.device(L.device):
        _lib.check(lib.fi_inside_backward(
            ctypes.byref(s), _p(L), _p(R), _p(root), _p(unary), _p(lengths), _p(log_z),
            _p(grad_log_z), _p(dL), _p(dR), _p(droot), _p(dunary), _p(ws), _stream(L.device)))
    return dL, dR, droot, dunary


@inside_bwd.register_fake
def _(grad_log_z, L, R, root, unary, lengths, log_z, ws, gemm_dtype, store_chart,
      chart_dtype="auto"):
    return (torch.empty_like(L), torch.empty_like(R), torch.empty_like(root),
            torch.empty_like(unary))


def _setup_context(ctx, inputs, output):
    L, R, root, unary, lengths, gemm_dtype, store_chart, chart_dtype = inputs
    log_z, ws = output
    ctx.save_for_backward(L, R, root, unary, lengths, log_z, ws)
    ctx.set_materialize_grads(False)  # never zero-fill a grad for the workspace output
    ctx.gemm_dtype = gemm_dtype
    ctx.store_chart = store_chart
    ctx.chart_dtype = chart_dtype


def _backward(ctx, grad_log_z, _grad_ws):
    L, R, root, unary, lengths, log_z, ws = ctx.saved_tensors
    dL, dR, droot, dunary = inside_bwd(grad_log_z, L, R, root, unary, lengths, log_z, ws,
                                       ctx.gemm_dtype, ctx.store_chart, ctx.chart_dtype)
    return dL, dR, droot, dunary, None, None, None, None


inside_fwd.register_autograd(_backward, setup_context=_setup_context)


def inside(L: torch.Tensor, R: torch.Tensor, root: torch.Tensor, unary: torch.Tensor,
           lengths: torch.Tensor, gemm_dtype: str = "bf16", chart_dtype: str = "auto",
           validate: bool = True) -> torch.Tensor:
    """Per-sentence log partition log Z (B,), differentiable in L, R, root, unary.

    gemm_dtype: "bf16" | "tf32" (fast modes, 2e-3 parity bound) or "fp32"
    (bf16x3 split operands, 1e-4 bound).  chart_dtype: storage of the
    projected chart vectors between GEMM and split kernels -- "auto" (fp16
    linear in the fast modes, fp32 log in fp32 mode), "fp32" or "fp16".
    validate: raise ValueError naming the first sentence whose length is
    outside [2, l] (one host read); with validate=False such a sentence gets
    log Z = NaN and no gradient (the device-side guard), for callers that
    check log Z themselves without a sync (TrainStep).  A zero-probability
    sentence returns log Z = -inf and contributes no gradient."""
    if validate:
        check_lengths(lengths, unary.shape[1] if unary.dim() == 3 else 0)
    log_z, _ = inside_fwd(L, R, root, unary, lengths, gemm_dtype, False, chart_dtype)
    return log_z


def inside_with_workspace(L, R, root, unary, lengths, gemm_dtype="bf16", store_chart=False,
                          chart_dtype="auto"):
    """Forward only, returning (log_z, workspace) for chart export / explicit backward."""
    check_lengths(lengths, unary.shape[1] if unary.dim() == 3 else 0)
    with torch.no_grad():
        return inside_fwd(L, R, root, unary, lengths, gemm_dtype, store_chart, chart_dtype)


def test_gemm(A: torch.Tensor, B: torch.Tensor, a_mn: bool = False, b_mn: bool = False
              ) -> torch.Tensor:
    """C = A_op @ B_op^T through the engine's tcgen05 GEMM (test hook).

    A is (M, K) (or (K, M) when a_mn), B is (N, K) (or (K, N) when b_mn);
    bf16 tensors use kind::f16, fp32 tensors use kind::tf32."""
    dtype = {torch.bfloat16: _lib.FI_GEMM_BF16, torch.float32: _lib.FI_GEMM_TF32}[A.dtype]
    M = A.shape[1] if a_mn else A.shape[0]
    K = A.shape[0] if a_mn else A.shape[1]
    N = B.shape[1] if b_mn else B.shape[0]
    C = torch.empty(M, N, dtype=torch.float32, device=A.device)
    lib = _lib.load()
    with torch.cuda.device(A.device):
        _lib.check(lib.fi_test_gemm(dtype, int(a_mn), int(b_mn), M, N, K, _p(A.contiguous()),
                                    _p(B.contiguous()), _p(C), _stream(A.device)))
    return C
