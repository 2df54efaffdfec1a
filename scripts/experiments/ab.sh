FI_CLUSTER=1 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
FI_CLUSTER=2 FI_BULK=0 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for cfg in "FI_BULK=0 FI_CLUSTER=1" "FI_BULK=0 FI_CLUSTER=2" "FI_BULK=0 FI_CLUSTER=4" "FI_BULK=1 FI_CLUSTER=1 FI_STAGES=4" "FI_BULK=1 FI_CLUSTER=2 FI_STAGES=4" "FI_BULK=1 FI_CLUSTER=2 FI_STAGES=6" "FI_BULK=1 FI_CLUSTER=4 FI_STAGES=3"; do
  env $cfg python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('$cfg', round(d['ms_per_step'],2), {k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in pc.items() if k in ('split_fwd','gather_bwd')})"
done
