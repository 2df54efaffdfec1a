# per-width A/B: build_ab/$1 vs the current build
echo "== ref $1"; FI_LIB_PATH=build_ab/$1 timeout 300 python scripts/per_width.py 2>&1 | tail -45
echo "== new"; timeout 300 python scripts/per_width.py 2>&1 | tail -45
