"""Host-side grammar types of the reference's engine interface.

Mirrors the pieces of /root/reference/pkg/src/flashpcfg/grammar.py that sit on
the inside-algorithm boundary, with the same names and semantics so that a
caller can hand either the reference's objects or these to the engine:

* GrammarDims      grammar.py:37-53   symbol / vocabulary counts, n_sym
* SimpleGrammar    grammar.py:62-108  frozen float64 log tables; tied L = R
* random_grammar   grammar.py:160-180 Dirichlet rows (same RNG draw order, so
                                      identical tables for identical seeds)
* GrammarGrad      grammar.py:357-392 gradient carrier (add_, scale_)

Everything here is NumPy bookkeeping; no compute of the hot path happens on
the host.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class GrammarError(Exception):
    """Structurally invalid grammar (shapes, flags, dims)."""


@dataclass(frozen=True)
class GrammarDims:
    n_nt: int
    n_pt: int
    vocab_size: int

    def __post_init__(self):
        for name in ("n_nt", "n_pt", "vocab_size"):
            val = getattr(self, name)
            if not isinstance(val, (int, np.integer)) or val < 1:
                raise GrammarError(f"{name} must be a positive integer, got {val!r}")

    @property
    def n_sym(self) -> int:
        return self.n_nt + self.n_pt


def _readonly(a) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    out.setflags(write=False)
    return out


@dataclass
class SimpleGrammar:
    """Log-space simple PCFG: root (N,), left/right (N, N+P), emit (P, V)."""

    dims: GrammarDims
    log_root: np.ndarray
    log_left: np.ndarray
    log_right: np.ndarray
    log_emit: np.ndarray
    tied: bool = False

    def __post_init__(self):
        self.log_root = _readonly(self.log_root)
        self.log_left = _readonly(self.log_left)
        self.log_right = self.log_left if self.tied else _readonly(self.log_right)
        self.log_emit = _readonly(self.log_emit)
        d = self.dims
        want = {"log_root": (d.n_nt,), "log_left": (d.n_nt, d.n_sym),
                "log_right": (d.n_nt, d.n_sym), "log_emit": (d.n_pt, d.vocab_size)}
        for name, shp in want.items():
            if getattr(self, name).shape != shp:
                raise GrammarError(
                    f"{name} has shape {getattr(self, name).shape}, expected {shp}")


def _dirichlet_log_rows(rng: np.random.Generator, rows: int, cols: int,
                        concentration: float) -> np.ndarray:
    probs = rng.dirichlet(np.full(cols, concentration), size=rows)
    with np.errstate(divide="ignore"):  # exact zeros become -inf log-probs
        return np.log(probs)


def random_grammar(dims: GrammarDims, seed: int, concentration: float = 1.0,
                   tied: bool = False) -> SimpleGrammar:
    """Dirichlet(concentration) rows drawn root, left, right, emit in that order."""
    if concentration <= 0:
        raise GrammarError(f"concentration must be > 0, got {concentration}")
    rng = np.random.default_rng(seed)
    root = _dirichlet_log_rows(rng, 1, dims.n_nt, concentration)[0]
    left = _dirichlet_log_rows(rng, dims.n_nt, dims.n_sym, concentration)
    right = left if tied else _dirichlet_log_rows(rng, dims.n_nt, dims.n_sym, concentration)
    emit = _dirichlet_log_rows(rng, dims.n_pt, dims.vocab_size, concentration)
    return SimpleGrammar(dims, root, left, right, emit, tied=tied)


@dataclass
class GrammarGrad:
    """d log_z / d (log-table entry), unconstrained; left/right kept separate."""

    d_root: np.ndarray
    d_left: np.ndarray
    d_right: np.ndarray
    d_emit: np.ndarray

    @classmethod
    def zeros(cls, dims: GrammarDims) -> "GrammarGrad":
        return cls(np.zeros(dims.n_nt), np.zeros((dims.n_nt, dims.n_sym)),
                   np.zeros((dims.n_nt, dims.n_sym)), np.zeros((dims.n_pt, dims.vocab_size)))

    def add_(self, other: "GrammarGrad") -> "GrammarGrad":
        for name in ("d_root", "d_left", "d_right", "d_emit"):
            getattr(self, name).__iadd__(getattr(other, name))
        return self

    def scale_(self, c: float) -> "GrammarGrad":
        for name in ("d_root", "d_left", "d_right", "d_emit"):
            getattr(self, name).__imul__(c)
        return self
