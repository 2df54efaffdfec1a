# thin-launch dual-stream sweep: parity under the dual paths, then step time per threshold
FI_DUAL_ROWS=100000000 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graph.py -q -x 2>&1 | tail -1
FI_DUAL_ROWS=768 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for r in 0 512 768 1152 1536 0 768 1152; do
  echo "rows=$r $(FI_DUAL_ROWS=$r timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python scripts/bj.py x)"
done
