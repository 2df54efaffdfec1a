"""bench.py's reference arm on the CPU, as the driver launches it: one JSON
line with the contract keys, alone and under torchrun (rank 0 prints)."""

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
        "cpu_baseline", "e2e"}


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def _check(d: dict):
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_single_process():
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1",
                          "--steps", "1", "--warmup", "1"], cwd=ROOT, capture_output=True,
                         text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    _check(_line(res.stdout))


def test_reference_arm_under_torchrun():
    res = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                          "--nproc-per-node", "2", "--master-addr", "127.0.0.1",
                          "--master-port", "29571", "bench.py", "--impl", "reference",
                          "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    d = _line(res.stdout)
    _check(d)
    assert d["n_gpus"] == 2


def test_gpus_flag_without_torchrun_launches_the_ranks():
    """`python bench.py --gpus 2` (no torchrun): bench relaunches itself under
    torch.distributed.run; one JSON line, n_gpus 2."""
    res = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2",
                          "--config", "1", "--steps", "1", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr[-2000:]
    d = _line(res.stdout)
    _check(d)
    assert d["n_gpus"] == 2
