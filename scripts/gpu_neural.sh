timeout 600 python -m pytest tests/test_gpu_neural.py -q -x --tb=short 2>&1 | tail -15
