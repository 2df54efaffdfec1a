echo "== gemm tests pair=1"; FI_GEMM_PAIR=1 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short 2>&1 | tail -4
echo "== gemm tests pair=0"; FI_GEMM_PAIR=0 timeout 300 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short 2>&1 | tail -2
timeout 600 python scripts/gemm_bn_sweep.py
for cfg in "FI_GEMM_PAIR=-1" "FI_GEMM_PAIR=0"; do
env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$cfg', round(d['ms_per_step'],2), round(d['value'],1), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items()})"
done
timeout 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -3
