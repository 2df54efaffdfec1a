#!/bin/bash
# Round-2 measurement: smoke, GPU tests, bench (both arms), ncu launch list and
# full ncu captures of the split (w=20), gather (m=20), forward / dgrad GEMM
# (w=10) and the first wgrad GEMM of a config-3 step.
mkdir -p gpurun_out
O=gpurun_out/r02f
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build()" > ${O}_build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > ${O}_gputests.log 2>&1; tail -2 ${O}_gputests.log
SECONDS=0
timeout 900 python bench.py > ${O}_bench.json 2> ${O}_bench.err
echo "bench wall ${SECONDS}s"; python scripts/bj.py final < ${O}_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > ${O}_bench_ref.json 2>&1; tail -c 300 ${O}_bench_ref.json
P='python scripts/profile_step.py --steps 2'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${O}_launches.csv $P > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/pick_launches.py ${O}_launches.csv 20 40 > ${O}_pick20.txt
python scripts/pick_launches.py ${O}_launches.csv 10 40 > ${O}_pick10.txt
cat ${O}_pick20.txt ${O}_pick10.txt
mkdir -p /tmp/ncu
cap() { timeout 900 ncu --set full --clock-control none --import-source on -s $2 -c 1 -o /tmp/ncu/prof_$1 $P > /dev/null 2>&1; echo "ncu $1 rc=$?";
        ncu -i /tmp/ncu/prof_$1.ncu-rep --page details --csv > ${O}_prof_$1_details.csv 2>/dev/null; }
cap split $(awk '$1=="split"{print $2}' ${O}_pick20.txt)
cap gather $(awk '$1=="gather"{print $2}' ${O}_pick20.txt)
cap gemm_fwd $(awk '$1=="gemm_fwd"{print $2}' ${O}_pick10.txt)
cap gemm_dgrad $(awk '$1=="gemm_dgrad"{print $2}' ${O}_pick10.txt)
W=$(python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r02f_launches.csv").read().splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
ki = rows[hi].index("Kernel Name")
seen, seq = set(), []
for r in rows[hi + 1:]:
    if len(r) > ki and r[0] not in seen:
        seen.add(r[0]); seq.append((int(r[0]), r[ki]))
half = [k for k in seq if "k_prep_weights" in k[1]][1][0]
print(next(k[0] for k in seq if k[0] >= half and "k_gemm<" in k[1] and ", 1, 1, 3," in k[1]))
PY
)
cap gemm_wgrad $W
python scripts/summarize_profiles.py --tag r02 --launches ${O}_launches.csv --reps /tmp/ncu/prof_*.ncu-rep \
  --split-width 20 --gather-width 20 --gemm-width 10 > ${O}_summary.log 2>&1; tail -3 ${O}_summary.log
cp profiles/r02_launches_summary.md profiles/r02_ncu_kernels.json profiles/ncu_traffic.json gpurun_out/ 2>/dev/null
du -sh gpurun_out
