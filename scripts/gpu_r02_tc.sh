#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_schedules.py tests/test_gpu_neural.py -q -x > gpurun_out/r02tc_tests.log 2>&1; tail -2 gpurun_out/r02tc_tests.log
bash scripts/gpu_ab.sh 3 r02tc_ab old new
FI_LIB_PATH=build_ab/new.so timeout 300 python scripts/gemm_stage_probe.py 2>/dev/null | cut -c1-200
