echo "== old"; FI_LIB_PATH=build_ab/old.so FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
for st in 4 5 7; do echo "== new stages $st"; FI_GEMM_STAGES=$st FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py; done
echo "== new bn512"; FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
