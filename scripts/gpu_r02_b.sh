#!/bin/bash
# round 2: remaining new parity tests, dp engine tests, the new bench (N=1 graph, N=2 gloo dry run), TF32 peak
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02b_build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_dp.py tests/test_gpu_baseline_configs.py -q -s -m gpu -k "dp or config4 or config5 or peaked or trained" --durations=10 > gpurun_out/r02b_tests.log 2>&1
timeout 300 python scripts/measure_tf32.py > gpurun_out/r02b_tf32.log 2>&1
cp profiles/measured_tf32.json gpurun_out/ 2>/dev/null
timeout 600 python bench.py > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
timeout 600 python bench.py --gpus 2 --steps 3 --no-e2e > gpurun_out/r02b_bench_n2.json 2> gpurun_out/r02b_bench_n2.err
tail -3 gpurun_out/r02b_tests.log
