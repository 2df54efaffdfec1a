#!/bin/bash
mkdir -p gpurun_out
out=gpurun_out/r02sm.jsonl; : > $out
timeout 200 python scripts/gemm_small_m.py >> $out 2>/dev/null
for pb in "0 64" "0 128" "0 256" "1 128" "1 256"; do set -- $pb
  for ks in 1 2 3 4 6 8; do
    FI_GEMM_PAIR=$1 FI_GEMM_BN=$2 FI_GEMM_KSPLIT=$ks FI_GEMM_NOTAIL=1 timeout 200 python scripts/gemm_small_m.py >> $out 2>/dev/null
  done
done
python - <<'PY'
import json, collections
rows = [json.loads(l) for l in open("gpurun_out/r02sm.jsonl") if l.startswith("{")]
best = collections.defaultdict(lambda: (1e9, ""))
dflt = {}
for r in rows:
    k = (r["kind"], r["M"])
    if r["tag"] == "": dflt[k] = r["us"]
    elif r["us"] == r["us"] and r["us"] < best[k][0]: best[k] = (r["us"], r["tag"])
for k in sorted(best):
    print(k, "default %.1f" % dflt.get(k, float("nan")), "best %.1f" % best[k][0], best[k][1])
PY
