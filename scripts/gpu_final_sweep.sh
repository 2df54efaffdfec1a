#!/bin/bash
# end-of-round bench lines of the secondary configurations (profiles/r02_bench_*.json)
mkdir -p gpurun_out/sweep
S=gpurun_out/sweep
run() { name=$1; shift; timeout 900 python bench.py --no-cpu-baseline "$@" > $S/r02_bench_$name.json 2>/dev/null; python scripts/bj.py "$name" < $S/r02_bench_$name.json | cut -c1-230; }
run cfg1 --config 1
run cfg2 --config 2
for l in 10 20 30 50 60; do run cfg4_l$l --length $l --no-e2e; done
run cfg5 --config 5
run cfg3_tf32 --gemm-dtype tf32
run cfg3_fp32 --gemm-dtype fp32
run cfg3_b8 --batch 8 --no-e2e
