python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; python -c "
import json; d=json.loads(open('gpurun_out/bench_r01.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['e2e'], d['clocks'])
print({k:(round(v['ms_per_step'],2), round(v.get('frac',0),3)) for k,v in d['roofline']['per_class'].items()})"; tail -3 gpurun_out/bench_r01.err
