"""Grammar (.spcfg) and parameter (.sprm) files: byte-compatible with the
reference's writers (tests/golden/ref_*, written by the reference) and
robust to corrupt input."""

from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2310_14997_b200 import formats, neural
from paper_2310_14997_b200.grammar import GrammarDims, random_grammar

GOLD = Path(__file__).parent / "golden"


@pytest.mark.parametrize("fname,dims,seed,tied", [("ref_untied.spcfg", (5, 4, 7), 11, False),
                                                   ("ref_tied.spcfg", (3, 6, 4), 12, True)])
def test_grammar_files_match_reference(tmp_path, fname, dims, seed, tied):
    ref = GOLD / fname
    g = formats.load_grammar(ref)
    mine = random_grammar(GrammarDims(*dims), seed=seed, tied=tied)
    assert g.tied == tied
    for k in ("log_root", "log_left", "log_right", "log_emit"):
        np.testing.assert_array_equal(getattr(g, k), getattr(mine, k))
    out = tmp_path / "g.spcfg"
    formats.save_grammar(mine, out)
    assert out.read_bytes() == ref.read_bytes()          # byte-identical to the reference


def test_param_file_matches_reference(tmp_path):
    ref = GOLD / "ref_params.sprm"
    p = formats.load_params(ref, dtype=torch.float64)
    mine = neural.init_params(GrammarDims(4, 3, 5), 6, 13, dtype=torch.float64)
    for k in mine.tensors:
        np.testing.assert_array_equal(p.tensors[k].numpy(), mine.tensors[k].numpy())
    out = tmp_path / "p.sprm"
    formats.save_params(mine, out)
    assert out.read_bytes() == ref.read_bytes()


def test_corrupt_grammar_files_name_the_field(tmp_path):
    data = (GOLD / "ref_untied.spcfg").read_bytes()
    cases = {"bad magic": b"XPCFG" + data[5:], "unsupported version": data[:5] + b"\x02" + data[6:],
             "unknown flag": data[:6] + b"\x04" + data[7:], "truncated while reading emission":
             data[:-8], "trailing bytes": data + b"\x00"}
    for msg, blob in cases.items():
        f = tmp_path / "x.spcfg"
        f.write_bytes(blob)
        with pytest.raises(formats.GrammarFileError, match=msg):
            formats.load_grammar(f)
    with pytest.raises(formats.GrammarFileError, match="cannot read"):
        formats.load_grammar(tmp_path / "missing.spcfg")


def test_corrupt_param_files(tmp_path):
    data = (GOLD / "ref_params.sprm").read_bytes()
    f = tmp_path / "x.sprm"
    for blob, msg in ((b"NOPE!" + data[5:], "bad magic"), (data[:-3], "truncated"),
                      (data + b"\x01", "trailing")):
        f.write_bytes(blob)
        with pytest.raises(formats.ParamFileError, match=msg):
            formats.load_params(f)
