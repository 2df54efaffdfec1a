# small-M GEMM shapes: default choice and forced (pair, bn, ksplit); FI_GEMM_INKERNEL_RED A/B
for red in 1 0; do
echo "red=$red default $(FI_GEMM_INKERNEL_RED=$red timeout 60 python scripts/gemm_small_m.py 2>&1 | tail -1)"
for p in 0 1; do for bn in 256; do for ks in 2 4 8; do
echo "red=$red pair=$p bn=$bn ks=$ks $(FI_GEMM_INKERNEL_RED=$red FI_GEMM_PAIR=$p FI_GEMM_BN=$bn FI_GEMM_KSPLIT=$ks FI_GEMM_NOTAIL=1 timeout 60 python scripts/gemm_small_m.py 2>&1 | tail -1)"
done; done; done; done
