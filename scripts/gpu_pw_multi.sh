# per-width totals for several builds in build_ab/ (same box)
for so in "$@"; do echo "== $so"; FI_LIB_PATH=build_ab/$so timeout 300 python scripts/per_width.py 2>&1 | tail -45; done
