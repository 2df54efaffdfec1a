#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_schedules.py -q -x -k "config3 or config2 or SPLIT_PERS or deep" > gpurun_out/r02m_tests.log 2>&1
tail -2 gpurun_out/r02m_tests.log
FI_LIB_PATH=build_ab/new.so timeout 300 python scripts/per_width.py > gpurun_out/r02m_perwidth_new.txt 2>&1
bash scripts/gpu_ab.sh 3 r02m_ab old new
