set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short -x -s -k "config2 or parity or config3" 2>&1 | grep -E "worst|passed|failed|Error|assert" | tail -30
timeout 900 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -5
for ch in auto fp32; do
timeout 600 python bench.py --steps 10 --warmup 3 --chart-dtype $ch --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$ch', round(d['ms_per_step'],2), round(d['value'],1), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items()})"
done
for cfg in "FI_CLUSTER=1" "FI_CLUSTER=4" "FI_STAGES=6" "FI_STAGES=8" "FI_GCLUSTER=2" "FI_GCLUSTER=8" "FI_GSTAGES=8" "FI_GSTAGES=10"; do
  env $cfg python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$cfg', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items() if k in ('split_fwd','gather_bwd')})"
done
