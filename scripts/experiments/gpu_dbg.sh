timeout 300 python -m pytest tests/test_gpu_engine.py -q -x --tb=long -k "survey_config_log_z and fp32" 2>&1 | grep -E "Error|error|assert|approx|==" | head -20
FI_NPROD=8 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -5
FI_PSTAGES=3 timeout 300 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -5
