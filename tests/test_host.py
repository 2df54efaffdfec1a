"""Host-side mirror of the reference interface: names, validation and error
behaviour that do not need a GPU (the GPU paths are in test_gpu_*.py)."""

import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2310_14997_b200 import engine, ops
from paper_2310_14997_b200.grammar import (GrammarDims, GrammarError, GrammarGrad,
                                           SimpleGrammar, random_grammar)

REF = Path("/root/reference/pkg/src")


@pytest.fixture
def g():
    return random_grammar(GrammarDims(3, 4, 5), seed=1)


def test_prepare_matches_reference_errors(g):
    with pytest.raises(engine.InsideError, match="length >= 2"):
        engine._prepare(g, np.array([0]))
    with pytest.raises(engine.InsideError, match="unknown token id 9"):
        engine._prepare(g, np.array([0, 9]))
    with pytest.raises(engine.InsideError):
        engine._prepare(g, np.zeros((2, 2), dtype=np.int64))
    assert engine._prepare(g, [1, 2, 3]).dtype == np.int64


def test_corpus_errors_carry_sentence_index(g):
    with pytest.raises(engine.InsideError, match="empty corpus"):
        engine.corpus_log_likelihood(g, [])
    with pytest.raises(engine.InsideError, match="unknown engine"):
        engine.corpus_log_likelihood(g, [[0, 1]], engine="nope")
    with pytest.raises(engine.InsideError, match="sentence 1"):
        engine.corpus_log_likelihood(g, [[0, 1], [0, 99]])


def test_registry_seam(g):
    reg = {"flash": object()}
    engine.register(reg)
    assert reg["b200"] is engine.inside_b200 and "flash" in reg
    assert engine.ENGINES["b200"] is engine.inside_b200


def test_op_refuses_cpu_tensors():
    L = torch.zeros(2, 4)
    with pytest.raises(ValueError, match="no CPU fallback"):
        ops._check_inputs(L, L, torch.zeros(2), torch.zeros(1, 3, 2),
                          torch.zeros(1, dtype=torch.int32))


def test_grammar_types():
    with pytest.raises(GrammarError):
        GrammarDims(0, 1, 1)
    d = GrammarDims(2, 3, 4)
    assert d.n_sym == 5
    g = random_grammar(d, seed=0, tied=True)
    assert g.log_left is g.log_right and not g.log_left.flags.writeable
    with pytest.raises(GrammarError):
        SimpleGrammar(d, np.zeros(2), np.zeros((2, 4)), np.zeros((2, 5)), np.zeros((3, 4)))
    gr = GrammarGrad.zeros(d)
    gr.d_left += 1.0
    gr.add_(gr).scale_(0.25)
    assert np.all(gr.d_left == 0.5)
    # Dirichlet rows are log-normalised
    assert np.allclose(np.exp(g.log_left).sum(1), 1.0)


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present")
def test_random_grammar_identical_to_reference():
    sys.path.insert(0, str(REF))
    from flashpcfg.grammar import GrammarDims as RD, random_grammar as rrg
    a = random_grammar(GrammarDims(7, 5, 9), seed=123, concentration=0.7)
    b = rrg(RD(7, 5, 9), seed=123, concentration=0.7)
    for name in ("log_root", "log_left", "log_right", "log_emit"):
        assert np.array_equal(getattr(a, name), getattr(b, name))


@pytest.mark.skipif(not REF.exists(), reason="reference tree not present")
def test_engine_registers_into_the_reference_registry():
    sys.path.insert(0, str(REF))
    import flashpcfg.inside as ref_inside
    reg = dict(ref_inside.ENGINES)
    engine.register(reg)
    assert set(reg) == set(ref_inside.ENGINES) | {"b200"}


def test_check_lengths_names_the_first_bad_sentence():
    """ops.check_lengths (the op's host-side refusal, inside.py:113-121) on
    CPU tensors: no GPU involved."""
    import torch
    from paper_2310_14997_b200.ops import check_lengths
    check_lengths(torch.tensor([2, 5, 5], dtype=torch.int32), 5)
    for lens, b in (([5, 1, 0], 1), ([6, 2, 3], 0), ([2, 3, -1], 2)):
        with pytest.raises(ValueError, match=f"sentence {b}: length"):
            check_lengths(torch.tensor(lens, dtype=torch.int32), 5)
