mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short -s -k "config2" 2>&1 | grep -E "worst|passed|failed|Error" | tail -12
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -3
for ch in auto fp32; do
timeout 600 python bench.py --steps 10 --warmup 3 --chart-dtype $ch --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$ch', round(d['ms_per_step'],2), round(d['value'],1), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items()})"
done
timeout 300 python scripts/per_width.py
