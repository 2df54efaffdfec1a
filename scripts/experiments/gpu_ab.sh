# A/B: build_ab/old.so (previous commit) vs the current build, same box
for i in 1 2; do
echo "== old"; FI_LIB_PATH=build_ab/old.so FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
echo "== new"; FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
done
