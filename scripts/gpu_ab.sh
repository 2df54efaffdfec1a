#!/bin/bash
# A/B of builds in build_ab/ on one box: "name[:ENV=V,...]" arguments, R rounds alternating
# usage: bash scripts/gpu_ab.sh ROUNDS OUTTAG spec1 spec2 ...
mkdir -p gpurun_out
rounds=$1; tag=$2; shift 2
for r in $(seq 1 $rounds); do
  for spec in "$@"; do
    so=${spec%%:*}; envs=""
    if [[ "$spec" == *:* ]]; then envs=$(echo ${spec#*:} | tr ',' ' '); fi
    line=$(env $envs FI_LIB_PATH=build_ab/$so.so timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 30 $BENCH_ARGS 2>/dev/null | python scripts/bj.py "$spec")
    echo "r$r $line" | tee -a gpurun_out/${tag}.txt
  done
done
