for i in 1 2 3; do for r in 1 0; do echo "red=$r $(FI_GEMM_INKERNEL_RED=$r timeout 300 python bench.py --no-e2e --no-cpu-baseline 2>/dev/null | python scripts/bj.py x | cut -c1-200)"; done; done
