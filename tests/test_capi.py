"""The C-ABI library: loads, exports every symbol include/flashinside.h
declares, and its host-side planning/validation behaves without a GPU."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2310_14997_b200 import _build, _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "flashinside.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\*?\s*(fi_[a-z_0-9]+)\s*\(", text, re.M)
    return sorted(set(names))


def test_header_declares_the_engine_entry_points():
    names = declared_functions()
    for must in ("fi_workspace_bytes", "fi_inside_forward", "fi_inside_backward",
                 "fi_marginals", "fi_last_error", "fi_get_chart_layout"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_functions():
        assert hasattr(lib, name), f"{name} declared in flashinside.h but not exported"
    # and the ctypes binding covers exactly the header
    bound = {n for n, _, _ in _lib.SIGNATURES}
    assert bound == set(declared_functions())


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", str(_build.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def rowbase(w, B, l):
    return B * ((w - 1) * (l + 1) - (w - 1) * w // 2)


@pytest.mark.parametrize("n,p,b,l,dt", [(4096, 4096, 64, 40, "bf16"), (1, 1, 1, 2, "fp32"),
                                        (100, 60, 5, 9, "tf32"), (1024, 1024, 32, 30, "bf16")])
def test_chart_layout_rows_and_padding(n, p, b, l, dt):
    s = _lib.shape(n, p, b, l, dt, store_chart=True)
    lay = _lib.chart_layout(s)
    assert lay.rows == rowbase(l, b, l) + b == b * l * (l + 1) // 2
    assert lay.np % 256 == 0 and lay.np >= n and lay.pp % 256 == 0 and lay.pp >= p
    assert lay.off_o >= 0
    nbytes = _lib.workspace_bytes(s)
    for off in (lay.off_a, lay.off_b, lay.off_o, lay.off_x, lay.off_lq, lay.off_flag):
        assert 0 <= off < nbytes and off % 1024 == 0
    # chart arrays do not overlap (a, b are fp16 in the fast modes' default chart)
    assert lay.chart_fmt == (_lib.FI_CHART_F32 if dt == "fp32" else _lib.FI_CHART_F16)
    esz_ab = 2 if lay.chart_fmt == _lib.FI_CHART_F16 else 4
    spans = {lay.off_a: esz_ab, lay.off_b: esz_ab, lay.off_o: 4, lay.off_lq: 4}
    offs = sorted(spans)
    assert all(offs[k] + spans[offs[k]] * lay.rows * lay.np <= offs[k + 1] for k in range(3))


@pytest.mark.parametrize("chart,fmt", [("auto", None), ("fp32", 1), ("fp16", 2)])
@pytest.mark.parametrize("dt", ["bf16", "tf32", "fp32"])
def test_chart_dtype_selects_storage(dt, chart, fmt):
    s = _lib.shape(256, 256, 4, 10, dt, True, chart)
    lay = _lib.chart_layout(s)
    if fmt is None:
        fmt = _lib.FI_CHART_F32 if dt == "fp32" else _lib.FI_CHART_F16
    assert lay.chart_fmt == fmt
    s32 = _lib.shape(256, 256, 4, 10, dt, True, "fp32")
    if fmt == _lib.FI_CHART_F16:   # a and b halve
        assert _lib.workspace_bytes(s32) - _lib.workspace_bytes(s) >= 4 * lay.rows * lay.np - 2048


def test_workspace_scales_and_store_chart_costs_a_chart():
    s0 = _lib.shape(1024, 1024, 8, 20, "bf16", False)
    s1 = _lib.shape(1024, 1024, 8, 20, "bf16", True)
    s2 = _lib.shape(1024, 1024, 8, 20, "fp32", False)
    assert _lib.workspace_bytes(s1) > _lib.workspace_bytes(s0)
    assert _lib.workspace_bytes(s2) > _lib.workspace_bytes(s0)   # hi + lo operand planes


@pytest.mark.parametrize("bad", [dict(n_nt=0), dict(n_pt=0), dict(batch=0), dict(max_len=1),
                                 dict(gemm_dtype=7), dict(chart_dtype=5)])
def test_invalid_shapes_are_rejected(bad):
    kw = dict(n_nt=8, n_pt=8, batch=2, max_len=5, gemm_dtype=0, store_chart=0, chart_dtype=0)
    kw.update(bad)
    s = _lib.FiShape(**kw)
    lib = _lib.load()
    assert lib.fi_workspace_bytes(ctypes.byref(s)) == 0
    rc = lib.fi_inside_forward(ctypes.byref(s), *([None] * 7), None)
    assert rc == _lib.FI_ERR_ARG
    assert lib.fi_last_error()


def test_null_pointers_are_rejected_before_touching_the_gpu():
    s = _lib.shape(8, 8, 2, 5)
    lib = _lib.load()
    rc = lib.fi_inside_forward(ctypes.byref(s), *([None] * 7), None)
    assert rc == _lib.FI_ERR_ARG
    assert b"null pointer" in lib.fi_last_error()
    with pytest.raises(_lib.EngineError):
        _lib.check(rc)


def test_version_and_launch_counter():
    lib = _lib.load()
    assert lib.fi_version() >= 1
    assert lib.fi_launch_count() >= 0


def test_workspace_grows_quadratically_in_length_and_linearly_in_batch():
    """The GPU counterpart of the reference's allocation-shape contract
    (tests/test_inside.py:174-187: the fused engine's memory grows ~l^2, not
    l^3): the engine's only memory is fi_workspace_bytes."""
    def ws(n, b, l):
        return _lib.workspace_bytes(_lib.shape(n, n, b, l, "bf16", False))
    for n in (64, 1024, 4096):
        r = (ws(n, 8, 48) - ws(n, 8, 2)) / (ws(n, 8, 24) - ws(n, 8, 2))
        assert r < 5.0, r                      # ~4 (l^2); cubic would be ~8
        r_b = (ws(n, 32, 24) - ws(n, 1, 24)) / (ws(n, 16, 24) - ws(n, 1, 24))
        assert 2.0 <= r_b < 2.1, r_b           # linear in the batch
    # and far below the reference's unfused O(l^3 N) split stack at cfg3
    l, n = 40, 4096
    assert ws(n, 1, l) < 8 * n * (l * (l + 1) * (l + 2) // 6)


def test_alloc_meter_api_matches_the_reference():
    from paper_2310_14997_b200.engine import AllocMeter
    m = AllocMeter()
    a = m.alloc((10, 4))
    b = m.alloc((3,), retained=True)
    assert m.transient_bytes == 320 and m.peak_transient_bytes == 320
    assert m.retained_bytes == b.nbytes == 24
    m.release(a)
    assert m.transient_bytes == 0 and m.peak_transient_bytes == 320
