#!/bin/bash
# B=8 per GPU (the strong-scaling load): GEMM choices and switch A/B
mkdir -p gpurun_out
export BENCH_ARGS="--batch 8"
FI_GEMM_LOG=1 FI_LIB_PATH=build_ab/cur.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 3 --warmup 3 --batch 8 2>&1 | grep "fi gemm" | sort | uniq -c | sort -rn > gpurun_out/b8_choices.txt
bash scripts/gpu_ab.sh 2 b8_ab cur cur:FI_GEMM_INKERNEL_RED=1 cur:FI_GEMM_MC=1 cur:FI_GEMM_TRANS=1 cur:FI_GEMM_FIXUP_US=4 cur:FI_GEMM_KSPLIT=1 cur:FI_GEMM_PAIR=0 cur:FI_GATHER_PERS=1
