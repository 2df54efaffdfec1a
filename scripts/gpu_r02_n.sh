#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_decode.py -q > gpurun_out/r02n_decode.log 2>&1
tail -3 gpurun_out/r02n_decode.log
timeout 300 python bench.py --batch 8 --no-e2e --no-cpu-baseline > gpurun_out/r02n_b8.json 2>/dev/null
python scripts/bj.py b8 < gpurun_out/r02n_b8.json
FI_GEMM_LOG=1 timeout 300 python scripts/per_width.py --batch 8 > gpurun_out/r02n_perwidth_b8.txt 2>&1
grep -v "fi gemm" gpurun_out/r02n_perwidth_b8.txt | head -50
