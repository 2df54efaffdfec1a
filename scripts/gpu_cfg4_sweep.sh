#!/bin/bash
# round 2: config 4 (|N| = 4096, l = 10..60, B = 64) and config 2 bench lines; config-5 fp32 parity
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c4_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_baseline_configs.py -q -s -k "config5" > gpurun_out/r02c4_cfg5tests.log 2>&1; grep -E "worst|passed|failed" gpurun_out/r02c4_cfg5tests.log
for l in 10 20 30 40 50 60; do
  timeout 600 python bench.py --length $l --no-e2e --no-cpu-baseline > gpurun_out/r02c4_l$l.json 2>/dev/null
  python scripts/bj.py "l=$l" < gpurun_out/r02c4_l$l.json | cut -c1-250
done
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r02c4_cfg2.json 2>/dev/null; python scripts/bj.py cfg2 < gpurun_out/r02c4_cfg2.json | cut -c1-250
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/r02c4_cfg1.json 2>/dev/null; python scripts/bj.py cfg1 < gpurun_out/r02c4_cfg1.json | cut -c1-250
