timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short 2>&1 | tail -2
timeout 600 python scripts/gemm_bn_sweep.py
for cfg in "FI_GEMM_PAIR=1" "FI_GEMM_PAIR=0"; do echo "== $cfg"; env $cfg timeout 300 python scripts/gemm_micro.py; done
