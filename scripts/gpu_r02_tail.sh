#!/bin/bash
mkdir -p gpurun_out
cat > /tmp/tail_probe.py <<'PY'
import sys, os, json, torch
sys.path.insert(0, '.')
from paper_2310_14997_b200.ops import test_gemm
def bench(f, n=20):
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): f()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
tag = ",".join(f"{k[8:]}={v}" for k, v in sorted(os.environ.items()) if k.startswith("FI_GEMM") and k != "FI_GEMM_LOG")
for kind in ("fwd", "dgrad"):
    for M in (2496, 2368, 1792, 1600, 1536, 1344, 1216, 1088, 960):
        N, K, bmn = (8192, 4096, False) if kind == "fwd" else (4096, 8192, True)
        A = torch.rand(M, K, device="cuda").bfloat16()
        B = (torch.rand(K, N, device="cuda") if bmn else torch.rand(N, K, device="cuda")).bfloat16()
        print(json.dumps({"tag": tag, "kind": kind, "M": M, "us": bench(lambda: test_gemm(A, B, False, bmn)) * 1e3}), flush=True)
PY
for cfg in "" "FI_GEMM_FIXUP_US=4 FI_GEMM_FIXUP_GBS=8000" "FI_GEMM_FIXUP_US=2 FI_GEMM_FIXUP_GBS=15000" "FI_GEMM_PAIR=1 FI_GEMM_BN=512"; do
  env $cfg FI_GEMM_LOG=1 timeout 300 python /tmp/tail_probe.py > /tmp/o.txt 2> /tmp/e.txt
  grep "^{" /tmp/o.txt >> gpurun_out/r02tail.jsonl; sort -u /tmp/e.txt | grep "fi gemm" >> gpurun_out/r02tail_choices.txt
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/r02tail.jsonl")]
t = collections.defaultdict(dict)
for r in rows: t[(r["kind"], r["M"])][r["tag"]] = r["us"]
tags = sorted({r["tag"] for r in rows})
print(tags)
for k in sorted(t): print(k, [round(t[k].get(g, float("nan")), 1) for g in tags])
PY
