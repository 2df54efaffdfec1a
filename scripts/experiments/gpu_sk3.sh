timeout 900 python -m pytest tests/test_gpu_gemm.py -q -x --tb=short 2>&1 | tail -3
for cfg in "FI_GEMM_SK=-1" "FI_GEMM_SK=0"; do
echo "== $cfg"; env $cfg timeout 300 python scripts/gemm_micro.py
env $cfg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$cfg', round(d['ms_per_step'],2), round(d['value'],1), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items()})"
env $cfg timeout 300 python scripts/per_width.py | tail -39 | awk '{print $1, $3, $6}' | tr '\n' ';'
echo
done
timeout 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -3
