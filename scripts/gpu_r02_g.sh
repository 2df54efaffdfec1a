#!/bin/bash
# round 2: coalesced split-K fixup: correctness + per-width + bench
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02g_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_schedules.py tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x -k "KSPLIT or gemm or config2 or config3" > gpurun_out/r02g_tests.log 2>&1
FI_GEMM_LOG=0 timeout 300 python scripts/per_width.py > gpurun_out/r02g_perwidth.txt 2>&1
timeout 600 python bench.py --no-e2e > gpurun_out/r02g_bench.json 2> gpurun_out/r02g_bench.err
tail -2 gpurun_out/r02g_tests.log; head -12 gpurun_out/r02g_perwidth.txt
python -c "import json; d=json.load(open('gpurun_out/r02g_bench.json')); print(d['ms_per_step'], d['value'])"
