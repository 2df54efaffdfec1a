timeout 900 python -m pytest tests -m gpu -q -x --tb=short 2>&1 | tail -2
for c in 3 2 1; do for pdl in 1 0; do
FI_PDL=$pdl timeout 300 python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); pc=d['roofline']['per_class']
print('cfg $c pdl $pdl', round(d['ms_per_step'],3), round(d['value'],1))"
done; done
