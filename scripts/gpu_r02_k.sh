#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02k_build.log 2>&1
for m in bf16 fp32; do
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"k_(gemm|pack|row|copy)" python scripts/prof_param.py $m 2>/dev/null | grep -v "^==" > gpurun_out/r02k_param_$m.csv
done
python - <<'PY'
import csv
for m in ("bf16", "fp32"):
    rows = list(csv.reader(open(f"gpurun_out/r02k_param_{m}.csv")))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); gi = h.index("Grid Size")
    data = rows[hi + 1:]
    n = len(data) // 4
    print(m, "last step:")
    for r in data[-n:]:
        print(f"  {float(r[vi])/1e3:8.1f} us  {r[gi]:14s} {r[ki][:90]}")
PY
