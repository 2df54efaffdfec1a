# Round-end measurement, part A: smoke, GPU tests, bench (both arms), ncu launch
# list, and full ncu captures of the split, gather and forward-GEMM launches.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -2
SECONDS=0
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench wall ${SECONDS}s"
python scripts/bj.py final < gpurun_out/bench_final.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_final_ref.json 2>&1; tail -c 300 gpurun_out/bench_final_ref.json
P='python scripts/profile_step.py --steps 2'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv $P > /dev/null 2>&1; echo "ncu list rc=$?"
python scripts/pick_launches.py gpurun_out/launches_final.csv 20 40 > gpurun_out/pick.txt; cat gpurun_out/pick.txt
cap() { timeout 900 ncu --set full --clock-control none --import-source on -s $2 -c 1 -o gpurun_out/prof_$1 $P > /dev/null 2>&1; echo "ncu $1 rc=$?"; }
cap split $(awk '$1=="split"{print $2}' gpurun_out/pick.txt)
cap gather $(awk '$1=="gather"{print $2}' gpurun_out/pick.txt)
python scripts/pick_launches.py gpurun_out/launches_final.csv 10 40 > gpurun_out/pick10.txt
cap gemm_fwd $(awk '$1=="gemm_fwd"{print $2}' gpurun_out/pick10.txt)
du -sh gpurun_out
