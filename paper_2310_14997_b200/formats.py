"""Grammar and parameter files of the reference, so the
engine consumes checkpoints written by the reference CLI and vice versa.

* ``.spcfg`` grammar container (grammar.py:426-478): magic ``SPCFG``,
  version 1, flags (bit 0 = tied), n_nt / n_pt / vocab_size as little-endian
  u64, then root, left, right (absent when tied) and emission tables as raw
  row-major little-endian float64.
* ``.sprm`` embedding-parameter checkpoint (neuralparam.py:410-461): magic
  ``SPRM1``, n_nt / n_pt / vocab / d / tensor count as u64, then per tensor
  its name (u64 length + UTF-8), rank (u64), shape (u64 each) and float64
  data, in the parameterisation's tensor order.

Both round-trip bit-exactly (float64 on disk; device tensors are cast on
load / save) and reject corrupt input naming the offending field.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np
import torch

from .grammar import GrammarDims, GrammarError, SimpleGrammar
from .neural import EmbeddingParams, ParamError, tensor_shapes

GRAMMAR_MAGIC = b"SPCFG"
GRAMMAR_VERSION = 1
PARAM_MAGIC = b"SPRM1"


class GrammarFileError(GrammarError):
    """Malformed grammar file (grammar.py:33-34)."""


class ParamFileError(ParamError):
    """Malformed parameter checkpoint (neuralparam.py:28-29)."""


class _Cursor:
    """Bounds-checked little-endian reader over a byte string."""

    def __init__(self, data: bytes, error: type[Exception]):
        self.data, self.pos, self.error = data, 0, error

    def bytes(self, n: int, what: str) -> bytes:
        end = self.pos + n
        if n < 0 or end > len(self.data):
            raise self.error(f"truncated while reading {what}")
        out, self.pos = self.data[self.pos:end], end
        return out

    def u64(self, what: str) -> int:
        return struct.unpack("<Q", self.bytes(8, what))[0]

    def f64(self, shape, what: str) -> np.ndarray:
        n = int(np.prod(shape, dtype=np.int64))
        return np.frombuffer(self.bytes(8 * n, what), dtype="<f8").reshape(shape).astype(np.float64)

    def end(self, what: str) -> None:
        if self.pos != len(self.data):
            raise self.error(f"{len(self.data) - self.pos} trailing bytes after {what}")


def _f64(a) -> bytes:
    if isinstance(a, torch.Tensor):
        a = a.detach().double().cpu().numpy()
    return np.ascontiguousarray(a, dtype="<f8").tobytes()


def save_grammar(g: SimpleGrammar, path) -> None:
    d = g.dims
    blob = [GRAMMAR_MAGIC, bytes([GRAMMAR_VERSION, 1 if g.tied else 0]),
            struct.pack("<3Q", d.n_nt, d.n_pt, d.vocab_size), _f64(g.log_root),
            _f64(g.log_left)]
    if not g.tied:
        blob.append(_f64(g.log_right))
    blob.append(_f64(g.log_emit))
    Path(path).write_bytes(b"".join(blob))


def load_grammar(path) -> SimpleGrammar:
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise GrammarFileError(f"cannot read grammar file: {e}") from e
    c = _Cursor(data, GrammarFileError)
    magic = c.bytes(len(GRAMMAR_MAGIC), "magic")
    if magic != GRAMMAR_MAGIC:
        raise GrammarFileError(f"bad magic {magic!r}, expected {GRAMMAR_MAGIC!r}")
    version = c.bytes(1, "version")[0]
    if version != GRAMMAR_VERSION:
        raise GrammarFileError(f"unsupported version {version}")
    flags = c.bytes(1, "flags")[0]
    if flags & ~1:
        raise GrammarFileError(f"unknown flag bits 0x{flags:02x}")
    n_nt, n_pt, vocab = c.u64("n_nt"), c.u64("n_pt"), c.u64("vocab_size")
    try:
        dims = GrammarDims(n_nt, n_pt, vocab)
    except GrammarError as e:
        raise GrammarFileError(str(e)) from e
    if n_nt * (n_nt + n_pt) > 1 << 32:
        raise GrammarFileError(f"implausible table size for dims {dims}")
    root = c.f64((n_nt,), "root table")
    left = c.f64((n_nt, dims.n_sym), "left table")
    tied = bool(flags & 1)
    right = left if tied else c.f64((n_nt, dims.n_sym), "right table")
    emit = c.f64((n_pt, vocab), "emission table")
    c.end("emission table")
    return SimpleGrammar(dims, root, left, right, emit, tied=tied)


def save_params(params: EmbeddingParams, path) -> None:
    d = params.dims
    blob = [PARAM_MAGIC, struct.pack("<5Q", d.n_nt, d.n_pt, d.vocab_size, params.d,
                                     len(params.tensors))]
    for name, t in params.tensors.items():
        raw = name.encode("utf-8")
        shape = tuple(t.shape)
        blob += [struct.pack("<Q", len(raw)), raw, struct.pack("<Q", len(shape)),
                 struct.pack(f"<{len(shape)}Q", *shape), _f64(t)]
    Path(path).write_bytes(b"".join(blob))


def load_params(path, device=None, dtype=torch.float32) -> EmbeddingParams:
    try:
        data = Path(path).read_bytes()
    except OSError as e:
        raise ParamFileError(f"cannot read parameter file: {e}") from e
    c = _Cursor(data, ParamFileError)
    if c.bytes(len(PARAM_MAGIC), "magic") != PARAM_MAGIC:
        raise ParamFileError("not a parameter checkpoint (bad magic)")
    n_nt, n_pt, vocab = c.u64("n_nt"), c.u64("n_pt"), c.u64("vocab_size")
    d, count = c.u64("embedding dim"), c.u64("tensor count")
    try:
        dims = GrammarDims(n_nt, n_pt, vocab)
    except GrammarError as e:
        raise ParamFileError(f"bad header dimensions: {e}") from e
    expected = tensor_shapes(dims, d)
    got: dict[str, np.ndarray] = {}
    for _ in range(count):
        nlen = c.u64("tensor name length")
        if nlen > 1 << 16:
            raise ParamFileError(f"implausible tensor name length {nlen}")
        name = c.bytes(nlen, "tensor name").decode("utf-8", errors="replace")
        rank = c.u64(f"rank of {name}")
        if rank > 8:
            raise ParamFileError(f"implausible rank {rank} for {name}")
        shape = tuple(c.u64(f"shape of {name}") for _ in range(rank))
        if name not in expected:
            raise ParamFileError(f"unknown tensor {name!r}")
        if shape != expected[name]:
            raise ParamFileError(f"tensor {name!r} has shape {shape}, expected {expected[name]}")
        got[name] = c.f64(shape, f"data of {name}")
    c.end("parameter checkpoint")
    missing = set(expected) - set(got)
    if missing:
        raise ParamFileError(f"checkpoint is missing tensors: {sorted(missing)}")
    return EmbeddingParams(dims, d, {k: torch.tensor(got[k], dtype=dtype, device=device)
                                     for k in expected})
