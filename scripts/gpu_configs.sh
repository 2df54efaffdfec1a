# other configurations for DESIGN's measured table
run() { echo "$* :: $(timeout 600 python bench.py --no-e2e --no-cpu-baseline "$@" 2>/dev/null | python scripts/bj.py x)"; }
run --config 5
run --gemm-dtype fp32
run --gemm-dtype tf32
run --config 2
for l in 10 20 30 50 60; do run --length $l; done
echo "train :: $(timeout 600 python bench.py --workload train --no-e2e --no-cpu-baseline 2>/dev/null | head -c 600)"
