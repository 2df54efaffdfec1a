"""Host-side decoder pieces against the reference (tests/golden/decode.npz)."""

from pathlib import Path

import numpy as np

from paper_2310_14997_b200.decode import sentence_f1, spans_from_splits

GOLD = np.load(Path(__file__).parent / "golden" / "decode.npz")


def spans(arr):
    return frozenset(map(tuple, arr.tolist()))


def test_sentence_f1_matches_reference():
    for k in range(int(GOLD["n_cases"])):
        l = int(GOLD[f"c{k}_meta"][4])
        got = sentence_f1(spans(GOLD[f"c{k}_mbr"]), spans(GOLD[f"c{k}_vit"]), l)
        assert got == float(GOLD[f"c{k}_f1_mbr_vs_vit"])


def test_sentence_f1_edge_cases():
    assert sentence_f1({(0, 2)}, {(0, 2)}, 2) == 1.0           # both filtered empty
    assert sentence_f1({(0, 3), (0, 2)}, {(0, 3)}, 3) == 0.0   # one side empty
    assert sentence_f1({(0, 4), (0, 2), (2, 4)}, {(0, 4), (0, 2), (1, 4)}, 4) == 0.5


def test_spans_from_splits_reads_a_right_branching_tree():
    l = 5
    split = np.zeros((l, l + 1), dtype=np.int32)
    for i in range(l):
        for j in range(i + 2, l + 1):
            split[i, j] = i + 1
    assert spans_from_splits(split, l) == frozenset((i, l) for i in range(l - 1))
