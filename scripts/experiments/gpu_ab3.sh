echo "== old"; FI_LIB_PATH=build_ab/old.so FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
echo "== new st4 bstride 32K"; FI_GEMM_BSTRIDE=32768 FI_GEMM_STAGES=4 FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
echo "== new st4"; FI_GEMM_STAGES=4 FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
echo "== new bn512 st4 bstride 48K"; FI_GEMM_BSTRIDE=49152 FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 FI_GEMM_STAGES=3 timeout 120 python scripts/gemm_epi_probe.py
