#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_parity.py -q -x -k "GATHER or config2 or config3 or long or zero" > gpurun_out/r02gp_tests.log 2>&1; tail -2 gpurun_out/r02gp_tests.log
FI_LIB_PATH=build_ab/new.so timeout 300 python scripts/per_width.py > gpurun_out/r02gp_perwidth.txt 2>&1
bash scripts/gpu_ab.sh 3 r02gp_ab new new:FI_GATHER_PERS=0 new:FI_GATHER_PERS=2
