# forced 256 x 512 pair tiles vs the default choice, engine GEMM vs cuBLAS
echo "== default"; timeout 120 python scripts/gemm_vs_cublas.py 2>&1
echo "== pair bn=512"; FI_GEMM_PAIR=1 FI_GEMM_BN=512 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_vs_cublas.py 2>&1
echo "== pair bn=384"; FI_GEMM_PAIR=1 FI_GEMM_BN=384 FI_GEMM_KSPLIT=1 timeout 120 python scripts/gemm_vs_cublas.py 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
FI_GEMM_PAIR=1 FI_GEMM_BN=512 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x 2>&1 | tail -3
