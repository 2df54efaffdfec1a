#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02l_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_neural.py tests/test_gpu_errors.py -q -x > gpurun_out/r02l_tests.log 2>&1
tail -2 gpurun_out/r02l_tests.log
bash scripts/gpu_r02_k.sh 2>&1 | tail -28
timeout 600 python bench.py --workload train > gpurun_out/r02l_bench_train.json 2> gpurun_out/r02l_bench_train.err
python scripts/bj.py train < gpurun_out/r02l_bench_train.json
