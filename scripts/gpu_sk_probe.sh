#!/bin/bash
# stream-K (FI_GEMM_STREAMK=2: forced wherever it fits) against whole tiles on dgrad shapes,
# plus the GEMM unit tests under forced stream-K
mkdir -p gpurun_out
FI_GEMM_STREAMK=2 FI_GEMM_TUNE=0 timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -1
for M in 1024 1600 2496; do
  FI_GEMM_TUNE=0 FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 60 python scripts/sk_probe.py $M 4096 8192
  FI_GEMM_TUNE=0 FI_GEMM_STREAMK=2 FI_GEMM_PAIR=1 FI_GEMM_BN=256 timeout 60 python scripts/sk_probe.py $M 4096 8192
done
