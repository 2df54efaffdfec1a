"""The engine's opt-in launch schedules (environment switches read once per
process, so each runs in a fresh interpreter) give the same results as the
default schedule: the oracle at a small size and, for the split-K / dual
paths, at |N| = 1024 against the float64 oracle."""

import json
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent

CHILD = r"""
import json, sys
import numpy as np
sys.path[:0] = ['.', 'tests']
from test_gpu_parity import make_case, run_op, rel_err
from oracle import flashinside_oracle as O
out = {}
for name, (N, P, V, B, lmax, seed, lengths) in {
        "small": (64, 64, 64, 8, 20, 0, None),
        "n1024": (1024, 1024, 64, 6, 14, 3, [14, 9, 14, 12, 5, 14])}.items():
    root, left, right, emit, unary, lens, _ = make_case(N, P, V, B, lmax, seed, lengths)
    grad = -np.ones(B) / B
    want = O.inside_batch(left, right, root, unary, lens, grad)
    got = run_op(root, left, right, unary, lens, grad, "bf16")
    out[name] = {k: rel_err(got[k], want[k]) for k in ("dL", "dR", "droot", "dunary")}
    out[name]["log_z"] = float(np.abs(got["log_z"] / want["log_z"] - 1).max())
print(json.dumps(out))
"""


@pytest.mark.parametrize("env", [
    {"FI_DUAL_ROWS": "48"},                       # narrow launches as two half-batch chains
    {"FI_DUAL": "1"},                             # every launch as two chains
    {"FI_GEMM_INKERNEL_RED": "1", "FI_GEMM_KSPLIT": "2"},  # split-K reduced in-kernel
    {"FI_GEMM_KSPLIT": "4"},                      # split-K through the fixup kernel
    {"FI_SPLIT_PERS": "0"},                       # one-shot split kernel at every width
    {"FI_SPLIT_PERS": "2"},                       # persistent split kernel at every width
    {"FI_SPLIT_WIDE": "0"},                       # widest spans with the plan's column split
    {"FI_PDL": "0"},
    {"FI_GATHER_PERS": "0"},                      # one-shot gather at every width
    {"FI_GATHER_PERS": "2"},                      # persistent gather at every width
    # multicast clusters (two CTA pairs sharing the A rows) for every eligible GEMM
    {"FI_GEMM_MC": "1", "FI_GEMM_PAIR": "1", "FI_GEMM_BN": "256", "FI_GEMM_KSPLIT": "1",
     "FI_GEMM_NOTAIL": "1"},
    {"FI_GEMM_MC": "1", "FI_GEMM_PAIR": "1", "FI_GEMM_BN": "128", "FI_GEMM_KSPLIT": "1",
     "FI_GEMM_NOTAIL": "1"},
    # transposed-output GEMMs (weight table on the MMA's M side) for fwd / dgrad / dunary
    {"FI_GEMM_TRANS": "1"},
    {"FI_GEMM_TRANS": "1", "FI_GEMM_KSPLIT": "3", "FI_GEMM_PAIR": "0"},
    {"FI_GEMM_TRANS": "1", "FI_GEMM_KSPLIT": "2", "FI_GEMM_PAIR": "1", "FI_GEMM_BN": "128"},
    {"FI_GEMM_TUNE": "0"},                        # the cost model's tile, never measured
    {"FI_GEMM_STREAMK": "2", "FI_GEMM_TUNE": "0"},  # stream-K tails wherever they fit
    {"FI_GEMM_TUNE_SPAN_PCT": "1000", "FI_GEMM_TUNE_MAX": "40"},  # time (run) many more tiles
], ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_schedule_matches_oracle(env):
    res = subprocess.run([sys.executable, "-c", CHILD], cwd=ROOT, capture_output=True, text=True,
                         env={**os.environ, **env}, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    errs = json.loads(res.stdout.strip().splitlines()[-1])
    for case, e in errs.items():
        for k, v in e.items():
            assert v < 2e-3, f"{env} {case} {k}: {v:.2e}"


def test_measured_tile_choice_is_reused():
    """The first eager launch of a GEMM shape times candidate tiles (FI_GEMM_TUNE,
    on by default); later launches of the shape reuse the stored pick, so a
    repeated call is bit-identical to the first."""
    sys.path[:0] = [str(ROOT), str(ROOT / "tests")]
    from test_gpu_parity import make_case, run_op
    root, left, right, emit, unary, lens, _ = make_case(1024, 1024, 64, 6, 14, 11, None)
    grad = -np.ones(6) / 6
    first = run_op(root, left, right, unary, lens, grad, "bf16")
    again = run_op(root, left, right, unary, lens, grad, "bf16")
    for k in first:
        assert np.array_equal(first[k], again[k]), k
