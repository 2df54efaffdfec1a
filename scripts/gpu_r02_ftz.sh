#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_baseline_configs.py tests/test_gpu_engine.py -q -x > gpurun_out/r02ftz_tests.log 2>&1; tail -2 gpurun_out/r02ftz_tests.log
bash scripts/gpu_ab.sh 3 r02ftz_ab old new
