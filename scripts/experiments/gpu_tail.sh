timeout 600 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short 2>&1 | tail -1
FI_GEMM_KSPLIT=3 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x --tb=short 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -1
for cfg in "FI_GEMM_NOTAIL=0" "FI_GEMM_NOTAIL=1"; do
env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python scripts/bj.py "$cfg"
done
env FI_GEMM_NOTAIL=0 timeout 300 python scripts/per_width.py | tail -39 | awk '{print $1, $3, $5, $7}' | tr '\n' ';'
