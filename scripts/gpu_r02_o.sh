#!/bin/bash
mkdir -p gpurun_out
for st in 3 4 5 6 7 9 12; do FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 FI_GEMM_STAGES=$st timeout 120 python scripts/gemm_stage_probe.py; done > gpurun_out/r02o_probe.jsonl 2>&1
for st in 2 3 4; do FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 FI_GEMM_STAGES=$st timeout 120 python scripts/gemm_stage_probe.py; done >> gpurun_out/r02o_probe.jsonl 2>&1
for st in 4 6 8 12; do FI_GEMM_PAIR=0 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 FI_GEMM_STAGES=$st timeout 120 python scripts/gemm_stage_probe.py; done >> gpurun_out/r02o_probe.jsonl 2>&1
cat gpurun_out/r02o_probe.jsonl | python -c "
import sys, json
for l in sys.stdin:
    if l.startswith('{'):
        d = json.loads(l); print(f\"{d['tag'][:80]:80s} {d['M']:5d} {d['us']:8.1f} {d['tflops']:7.1f}\")"
