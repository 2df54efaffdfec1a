timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -c 300
timeout 600 python bench.py --workload train --steps 5 --warmup 3 2>&1 | tail -c 1500
