for so in build_ab/old.so paper_2310_14997_b200/_flashinside.so; do echo "== $so"; FI_LIB_PATH=$so FI_GEMM_PAIR=1 FI_GEMM_BN=256 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py; done
echo "== bn512"; FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py
