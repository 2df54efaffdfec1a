#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/r02mc2.jsonl; : > $out
for mc in 0 1; do for bn in 64 128 256; do
  FI_GEMM_MC=$mc FI_GEMM_PAIR=1 FI_GEMM_BN=$bn FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 timeout 200 python scripts/gemm_small_m.py >> $out 2>/dev/null
done; done
python - <<'PY'
import json
rows = [json.loads(l) for l in open("gpurun_out/r02mc2.jsonl") if l.startswith("{")]
for r in rows:
    if r["M"] in (256, 448, 576): print(r["tag"], r["kind"], r["M"], round(r["us"], 1))
PY
