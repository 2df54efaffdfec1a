"""bench.py's algorithmic-work accounting (the roofline numerators) against
the closed forms of SURVEY §8(d), and its clock-sample filtering."""

import math
import time

import pytest

import bench


def test_forward_gemm_flops_match_survey():
    # F = 4 N P l + 4 N^2 (l(l-1)/2 - 1) per sentence, cfg3 54.96 GFLOP
    n = p = 4096
    l, b = 40, 64
    work = bench.algorithmic_work(n, p, b, l, 2, False, 2)
    f = 4 * n * p * l + 4 * n * n * (l * (l - 1) // 2 - 1)
    assert work["gemm_fwd"] == ("tensor", pytest.approx(b * f))
    assert f / 1e9 == pytest.approx(54.96, rel=1e-3)
    assert work["gemm_dgrad"][1] == work["gemm_wgrad"][1] == work["gemm_fwd"][1]


@pytest.mark.parametrize("esz", [2, 4])
def test_split_bytes_closed_form(esz):
    # every (span, split) pair reads two distinct rows: 2 s N C(l+1, 3) per
    # sentence, plus one E row per span below the top width
    n, b, l = 1024, 3, 30
    total = sum(bench.split_launch_bytes(n, b, l, w, 2, esz) for w in range(2, l + 1))
    reads = 2 * esz * n * math.comb(l + 1, 3) * b
    e_rows = sum(l - w + 1 for w in range(2, l)) * b * n * 2
    assert total == pytest.approx(reads + e_rows)


def test_gather_bytes_cover_every_wider_span():
    # child width m: 2 a/b rows + 1 outside-weight row per span wider than m,
    # plus the child's own a, b rows and its 2N-wide G row
    n, b, l, m = 256, 2, 10, 3
    s_m = (l - m) * (l - m + 1) // 2
    n_m = l - m + 1
    got = bench.gather_launch_bytes(n, b, l, m, 2, 4)
    assert got == pytest.approx(b * (s_m * n * (2 * 4 + 4) + n_m * (2 * n * 4 + 2 * n * 2)))
    # fp16 chart: 2-byte rows and one fp32 exponent per 32 outside weights
    got_h = bench.gather_launch_bytes(n, b, l, m, 2, 2)
    assert got_h == pytest.approx(b * (s_m * n * (2 * 2 + 2 + 4 / 32) + n_m * (2 * n * 2 + 2 * n * 2)))


def test_clock_sampler_keeps_only_timed_region_lines():
    cs = bench.ClockSampler(0)
    cs.proc = None
    now = time.time()
    line = "2026/10/17 10:00:00.000, {sm}, 1965, 700.0, Not Active, Not Active, Not Active, {cap}"
    cs.lines = [(now - 5.0, line.format(sm=120, cap="Not Active")),   # warm-up: dropped
                (now - 0.01, line.format(sm=1900, cap="Active")),
                (now, line.format(sm=1950, cap="Not Active"))]
    cs.t_mark = now - 1.0

    class _P:  # a finished nvidia-smi process
        def terminate(self):
            pass

        def wait(self, timeout=None):
            return 0

    cs.proc = _P()
    out = cs.stop()
    assert out["samples"] == 2
    assert out["sm_mhz"] == pytest.approx(1925.0)
    assert out["sm_max_mhz"] == 1965.0
    assert out["reasons"] == ["sw_power_cap"]
