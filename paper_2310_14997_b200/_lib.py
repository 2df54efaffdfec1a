"""ctypes binding of the C ABI in include/flashinside.h.

Loading fails loudly: there is no CPU fallback for the engine.  The
signatures mirror the header one for one; this module is also the model for
the reference-side binding shown in INTEGRATION.md.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, Structure, c_float, c_int32, c_int64, c_size_t, c_void_p, c_char_p

from . import _build

FI_OK = 0
FI_ERR_ARG = 1
FI_ERR_CUDA = 2
FI_ERR_UNSUPPORTED = 3
FI_GEMM_BF16 = 0
FI_GEMM_TF32 = 1
FI_GEMM_FP32 = 2
FI_CHART_AUTO = 0
FI_CHART_F32 = 1
FI_CHART_F16 = 2
FI_FLAG_ZERO_PROB = 1
FI_FLAG_BAD_LENGTH = 2

PROF_CLASSES = ("prep", "split_fwd", "gemm_fwd", "seed", "gather_bwd", "gemm_dgrad",
                "gemm_wgrad", "param")

GEMM_DTYPES = {"bf16": FI_GEMM_BF16, "tf32": FI_GEMM_TF32, "fp32": FI_GEMM_FP32}
CHART_DTYPES = {"auto": FI_CHART_AUTO, "fp32": FI_CHART_F32, "fp16": FI_CHART_F16}


class FiShape(Structure):
    _fields_ = [
        ("n_nt", c_int32),
        ("n_pt", c_int32),
        ("batch", c_int32),
        ("max_len", c_int32),
        ("gemm_dtype", c_int32),
        ("store_chart", c_int32),
        ("chart_dtype", c_int32),
    ]


class FiChartLayout(Structure):
    _fields_ = [
        ("np", c_int64),
        ("pp", c_int64),
        ("rows", c_int64),
        ("off_a", c_int64),
        ("off_b", c_int64),
        ("off_o", c_int64),
        ("off_x", c_int64),
        ("off_lq", c_int64),
        ("off_flag", c_int64),
        ("chart_fmt", c_int64),
        ("off_lqs", c_int64),
    ]


# (name, restype, argtypes) exactly as declared in include/flashinside.h
_PF = POINTER(c_float)
SIGNATURES = [
    ("fi_workspace_bytes", c_size_t, [POINTER(FiShape)]),
    ("fi_get_chart_layout", c_int32, [POINTER(FiShape), POINTER(FiChartLayout)]),
    ("fi_inside_forward", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p]),
    ("fi_inside_backward", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_inside_backward_ex", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_marginals", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_span_marginals", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_mbr_decode", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_viterbi", c_int32,
     [POINTER(FiShape), c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_param_workspace_bytes", c_size_t, [c_int32, c_int32, c_int32, c_int32]),
    ("fi_param_scores", c_int32,
     [c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    ("fi_param_scores_backward", c_int32,
     [c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
      c_void_p, c_void_p, c_void_p]),
    ("fi_test_gemm", c_int32,
     [c_int32, c_int32, c_int32, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p,
      c_void_p]),
    ("fi_launch_count", c_int64, []),
    ("fi_profile_enable", None, [c_int32]),
    ("fi_profile_collect", c_int32, [POINTER(c_float), POINTER(c_int32), c_int32]),
    ("fi_profile_collect_launches", c_int32, [POINTER(c_float), POINTER(c_int32), c_int32]),
    ("fi_last_error", c_char_p, []),
    ("fi_version", c_int32, []),
]

_LIB = None


class EngineError(RuntimeError):
    """A C-ABI call returned an error code."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"flashinside error {code}: {msg}")
        self.code = code


def load(build_if_missing: bool = True) -> ctypes.CDLL:
    """Load (building first if needed) the engine library; raise if impossible."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_missing and _build.needs_build():
        _build.build()
    if not _build.LIB_PATH.exists():
        raise RuntimeError(f"FlashInside engine library missing: {_build.LIB_PATH} "
                           "(run __graft_entry__.build()); there is no CPU fallback")
    # FI_LIB_PATH: load another build of the same C ABI (A/B timing runs)
    lib = ctypes.CDLL(os.environ.get("FI_LIB_PATH") or str(_build.LIB_PATH))
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def check(code: int) -> None:
    if code != FI_OK:
        msg = load().fi_last_error()
        raise EngineError(code, msg.decode() if msg else "")


def shape(n_nt: int, n_pt: int, batch: int, max_len: int, gemm_dtype: str = "bf16",
          store_chart: bool = False, chart_dtype: str = "auto") -> FiShape:
    if gemm_dtype not in GEMM_DTYPES:
        raise ValueError(f"gemm_dtype must be one of {sorted(GEMM_DTYPES)}, got {gemm_dtype!r}")
    if chart_dtype not in CHART_DTYPES:
        raise ValueError(f"chart_dtype must be one of {sorted(CHART_DTYPES)}, got {chart_dtype!r}")
    return FiShape(int(n_nt), int(n_pt), int(batch), int(max_len), GEMM_DTYPES[gemm_dtype],
                   1 if store_chart else 0, CHART_DTYPES[chart_dtype])


def workspace_bytes(s: FiShape) -> int:
    n = load().fi_workspace_bytes(ctypes.byref(s))
    if n == 0:
        check(FI_ERR_ARG)
    return int(n)


def chart_layout(s: FiShape) -> FiChartLayout:
    out = FiChartLayout()
    check(load().fi_get_chart_layout(ctypes.byref(s), ctypes.byref(out)))
    return out


def profile_enable(on: bool) -> None:
    load().fi_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    """{class: (total_ms, launches)} since the last collect (synchronizes)."""
    n = len(PROF_CLASSES)
    ms = (c_float * n)()
    cnt = (c_int32 * n)()
    check(load().fi_profile_collect(ms, cnt, n))
    return {name: (float(ms[i]), int(cnt[i])) for i, name in enumerate(PROF_CLASSES)}


def profile_collect_launches(max_launches: int = 65536) -> list[tuple[str, float]]:
    """[(class, ms)] per recorded launch in issue order (synchronizes, clears)."""
    ms = (c_float * max_launches)()
    cls = (c_int32 * max_launches)()
    k = load().fi_profile_collect_launches(ms, cls, max_launches)
    return [(PROF_CLASSES[cls[i]], float(ms[i])) for i in range(min(k, max_launches))]
