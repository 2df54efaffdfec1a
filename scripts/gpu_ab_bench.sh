# step-time A/B of builds in build_ab/ (bench.py graph replay, alternating)
for so in "$@"; do echo "$so $(FI_LIB_PATH=build_ab/$so timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python scripts/bj.py x)"; done
