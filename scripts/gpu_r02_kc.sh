#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -q -x -k "config or gemm or deep" > gpurun_out/r02kc_tests.log 2>&1; tail -2 gpurun_out/r02kc_tests.log
bash scripts/gpu_ab.sh 3 r02kc_ab old new
