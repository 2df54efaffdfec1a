"""dgrad-shaped GEMMs (N = 4096, K = 8192) with MN-major B (the W table
read untransposed, as the engine's dgrad does) against K-major B, and the
forward shape (N = 8192, K = 4096) for comparison (test hook, EPI_STORE,
measured tile choice)."""
import json
import sys

import torch

sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm  # noqa: E402


def bench(f, n=20):
    for _ in range(3):
        f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        f()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


import argparse
ap = argparse.ArgumentParser()
ap.add_argument("--all", action="store_true", help="every config-3 dgrad M (64 x 2..39)")
a = ap.parse_args()
tot = {}
for M in ([64 * (41 - w) for w in range(3, 41)] if a.all else (128, 640, 1280, 1920, 2496)):
    rec = {"M": M}
    for name, N, K, bmn in (("dgrad_mn", 4096, 8192, True), ("dgrad_k", 4096, 8192, False),
                            ("fwd_k", 8192, 4096, False)):
        A = torch.rand(M, K, device="cuda").bfloat16()
        Bm = (torch.rand(K, N, device="cuda") if bmn else torch.rand(N, K, device="cuda")).bfloat16()
        us = bench(lambda: test_gemm(A, Bm, False, bmn))
        rec[name] = round(us, 1)
        rec[name + "_tf"] = round(2 * M * N * K / us / 1e6, 0)
    print(json.dumps(rec), flush=True)
    for k in ("dgrad_mn", "dgrad_k", "fwd_k"):
        tot[k] = tot.get(k, 0.0) + rec[k]
    tot["best_of_mn_k"] = tot.get("best_of_mn_k", 0.0) + min(rec["dgrad_mn"], rec["dgrad_k"])
print(json.dumps({"total_us": {k: round(v, 1) for k, v in tot.items()}}))
