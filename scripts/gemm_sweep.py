"""Per-shape GEMM timing of the engine's tcgen05 GEMM (test hook, EPI_STORE)
on the config-3 step shapes, under the tile choice forced by the FI_GEMM_*
environment of this process (run once per setting), next to cuBLAS.

    FI_GEMM_PAIR=1 FI_GEMM_BN=384 python scripts/gemm_sweep.py --tag p1bn384
"""
import argparse
import json
import sys

import torch

sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--tag", default="default")
ap.add_argument("--cublas", action="store_true")
ap.add_argument("--batch", type=int, default=64)
a = ap.parse_args()


def bench(f, n=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


l, B = 40, a.batch
out = []
for kind in ("fwd", "dgrad"):
    for w in (1, 2, 3, 4, 5, 6, 8, 10, 12, 15, 18, 20, 23, 25, 28, 30, 32, 34, 35, 36, 37, 38, 39):
        M = B * (l - w + 1) if w > 1 else B * l
        if kind == "fwd":
            N, K, bmn = 8192, 4096, False
        else:
            N, K, bmn = 4096, 8192, True
        A = torch.rand(M, K, device="cuda").bfloat16()
        Bm = (torch.rand(K, N, device="cuda") if bmn else torch.rand(N, K, device="cuda")).bfloat16()
        try:
            ms = bench(lambda: test_gemm(A, Bm, False, bmn))
        except Exception as e:  # noqa: BLE001
            ms = float("nan")
            print(kind, w, "error", e, file=sys.stderr)
        rec = {"tag": a.tag, "kind": kind, "w": w, "M": M, "N": N, "K": K, "us": ms * 1e3}
        if a.cublas:
            Bt = Bm if bmn else Bm.t()
            rec["cublas_us"] = bench(lambda: torch.matmul(A, Bt)) * 1e3
        rec["ideal_us"] = 2 * M * N * K / 1.6663e15 * 1e6
        out.append(rec)
        print(json.dumps(rec), flush=True)
