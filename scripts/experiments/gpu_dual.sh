timeout 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -3
for cfg in "FI_DUAL=1" "FI_DUAL=0" "FI_DUAL=1 FI_DUAL_GEMM_STAGES=2" "FI_DUAL=1 FI_DUAL_GEMM_STAGES=4"; do
env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$cfg', round(d['ms_per_step'],2), round(d['value'],1), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items()})"
done
