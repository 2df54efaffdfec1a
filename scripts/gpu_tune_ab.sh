#!/bin/bash
# measured GEMM tile choice (FI_GEMM_TUNE) A/B at config 3 (B=64) and B=8
mkdir -p gpurun_out
bash scripts/gpu_ab.sh 3 tune_ab2_b64 tune:FI_GEMM_TUNE=0 tune:FI_GEMM_TUNE_SPAN_PCT=135,FI_GEMM_TUNE_MAX=8 tune tune:FI_GEMM_TUNE_SPAN_PCT=220,FI_GEMM_TUNE_MAX=16
BENCH_ARGS="--batch 8" bash scripts/gpu_ab.sh 2 tune_ab2_b8 tune:FI_GEMM_TUNE=0 tune tune:FI_GEMM_TUNE_SPAN_PCT=220,FI_GEMM_TUNE_MAX=16
