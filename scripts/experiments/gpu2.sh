timeout 600 python -m pytest tests/test_gpu_gemm.py -q --tb=line 2>&1 | tail -15
timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=short 2>&1 | grep -E "Error|passed|failed|worst|DESIRED|ACTUAL|Max rel" | head -60
