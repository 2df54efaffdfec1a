#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02j_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_neural.py tests/test_gpu_errors.py tests/test_gpu_reference_callers.py -q -x > gpurun_out/r02j_tests.log 2>&1
timeout 600 python bench.py --workload train > gpurun_out/r02j_bench_train.json 2> gpurun_out/r02j_bench_train.err
tail -3 gpurun_out/r02j_tests.log
python -c "import json; d=json.load(open('gpurun_out/r02j_bench_train.json')); print(d['ms_per_step'], d['value'], d['inside_engine_ms_per_step'], d['parameterisation_and_optimizer_ms_per_step'])"
