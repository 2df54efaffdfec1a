#!/bin/bash
# round 2, first GPU call: new parity/error tests, full gpu suite, bench
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_errors.py tests/test_gpu_baseline_configs.py -x -q -s -m gpu --durations=15 > gpurun_out/r02a_newtests.log 2>&1
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 1500 python -m pytest tests -q -m gpu --durations=20 --deselect tests/test_gpu_baseline_configs.py --deselect tests/test_gpu_errors.py > gpurun_out/r02a_gpusuite.log 2>&1
tail -3 gpurun_out/r02a_newtests.log gpurun_out/r02a_gpusuite.log
cat gpurun_out/r02a_bench.json | head -c 600
