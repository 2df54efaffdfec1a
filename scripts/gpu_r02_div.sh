#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedules.py tests/test_gpu_engine.py -q -x > gpurun_out/r02div_tests.log 2>&1; tail -2 gpurun_out/r02div_tests.log
bash scripts/gpu_ab.sh 3 r02div_ab old new
