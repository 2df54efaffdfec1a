run() { echo "== $*"; env "$@" timeout 300 python scripts/per_width.py 2>&1 | grep -A41 "^w "; }
run FI_STAGES=4
run FI_STAGES=8
run FI_STAGES=12
run FI_GSTAGES=10
