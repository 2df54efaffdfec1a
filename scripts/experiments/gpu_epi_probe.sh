for bn in 256 512; do echo "== pair bn=$bn"; FI_GEMM_PAIR=1 FI_GEMM_BN=$bn FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_epi_probe.py; done
FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 timeout 300 ncu --set full --clock-control none -k regex:k_gemm -s 2 -c 1 -o gpurun_out/big512 python scripts/gemm_one.py 8192 8192 8192 > /dev/null 2>&1
