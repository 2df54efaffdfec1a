#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dp.py -q > gpurun_out/r02hs_tests.log 2>&1; tail -2 gpurun_out/r02hs_tests.log
for r in 1 2; do timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02hs_bench$r.json 2>/dev/null
python -c "import json; d=json.loads([l for l in open('gpurun_out/r02hs_bench$r.json') if l.startswith('{')][-1]); print('device', round(d['ms_per_step'],2), round(d['value'],1), 'e2e', round(d['e2e']['ms_per_step'],2), round(d['e2e']['value'],1))"; done
timeout 600 python bench.py --gpus 2 --steps 3 --no-other-scaling > gpurun_out/r02hs_n2.json 2>/dev/null; python -c "import json; d=json.loads([l for l in open('gpurun_out/r02hs_n2.json') if l.startswith('{')][-1]); print('n2', d['n_gpus'], d['e2e']['value'])"
