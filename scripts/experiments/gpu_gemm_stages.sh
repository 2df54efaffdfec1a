for st in 4 5 7 12; do echo "== stages $st"; FI_GEMM_STAGES=$st timeout 120 python scripts/gemm_vs_cublas.py 2>&1; done
