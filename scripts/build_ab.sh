#!/bin/bash
# build the engine library of git revision $1 into build_ab/$2.so (A/B timing via FI_LIB_PATH)
set -e
rev=$1; name=$2
d=$(mktemp -d)
git archive "$rev" paper_2310_14997_b200/csrc include | tar -x -C "$d"
mkdir -p build_ab
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared --expt-relaxed-constexpr -o build_ab/$name.so "$d/paper_2310_14997_b200/csrc/fi_capi.cu"
rm -rf "$d"
echo built build_ab/$name.so from $rev
