cp paper_2310_14997_b200/_flashinside.so /tmp/c8.so
for c in 8 16 32; do
  if [ $c != 8 ]; then cp paper_2310_14997_b200/_flashinside_c$c.so paper_2310_14997_b200/_flashinside.so; fi
  echo "== chunk $c"
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_engine.py -q -x -s -k "fp32 or config2" 2>&1 | grep -E "worst|passed|failed" | grep -E "fp32|passed|failed"
  timeout 600 python bench.py --gemm-dtype fp32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python scripts/bj.py "fp32 chunk $c"
done
cp /tmp/c8.so paper_2310_14997_b200/_flashinside.so
