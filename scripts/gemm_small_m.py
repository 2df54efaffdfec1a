"""Small-M GEMM shapes of the config-3 (and B = 8) step under this process's
forced FI_GEMM_* tile (one JSON line per shape)."""
import json, os, sys
import torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm

def bench(f, n=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n

tag = ",".join(f"{k[8:]}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FI_GEMM"))
for kind in ("fwd", "dgrad"):
    for M in (128, 192, 256, 320, 448, 576, 704):
        N, K, bmn = (8192, 4096, False) if kind == "fwd" else (4096, 8192, True)
        A = torch.rand(M, K, device="cuda").bfloat16()
        B = (torch.rand(K, N, device="cuda") if bmn else torch.rand(N, K, device="cuda")).bfloat16()
        try:
            us = bench(lambda: test_gemm(A, B, False, bmn)) * 1e3
        except Exception as e:  # noqa: BLE001
            us = float("nan")
        print(json.dumps({"tag": tag, "kind": kind, "M": M, "us": us}), flush=True)
