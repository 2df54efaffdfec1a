timeout 600 python -m pytest tests/test_gpu_gemm.py -q --tb=line 2>&1 | tail -5
timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=short 2>&1 | grep -E "Error|passed|failed|worst|DESIRED|ACTUAL|Max rel|^FAILED" | head -60
timeout 300 python scripts/probe_perf.py 2>&1 | tail -20
