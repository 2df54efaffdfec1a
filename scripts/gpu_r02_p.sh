#!/bin/bash
mkdir -p gpurun_out
for mc in 0 1; do for st in 4 7; do FI_GEMM_LOG=1 FI_GEMM_MC=$mc FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 FI_GEMM_NOTAIL=1 FI_GEMM_STAGES=$st timeout 120 python scripts/gemm_stage_probe.py 2>&1 | grep -v "EPI=" | sort -u; done; done > gpurun_out/r02p_probe.txt
cat gpurun_out/r02p_probe.txt | cut -c1-200
