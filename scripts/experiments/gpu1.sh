set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q 2>&1 | tail -30
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -40
timeout 300 python scripts/probe_perf.py 2>&1 | tail -20
