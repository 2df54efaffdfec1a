# per-width split / gather times under decomposition overrides
run() { echo "== $*"; env "$@" timeout 300 python scripts/per_width.py 2>&1 | grep -A41 "^w "; }
run FI_SPLIT_PERS=1
run FI_SPLIT_PERS=0 FI_CLUSTER=1
run FI_SPLIT_PERS=0 FI_CLUSTER=2
run FI_SPLIT_PERS=0 FI_CLUSTER=4
run FI_SPLIT_PERS=0 FI_CLUSTER=8
run FI_GCLUSTER=1
run FI_GCLUSTER=4
run FI_GCLUSTER=8
