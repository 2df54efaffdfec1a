mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; tail -c 3000 gpurun_out/bench_r01.json; tail -5 gpurun_out/bench_r01.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu list rc=$?"; wc -l gpurun_out/launches_r01.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 180 -c 2 -o gpurun_out/prof_split python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 50 -c 2 -o gpurun_out/prof_gather python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 100 -c 3 -o gpurun_out/prof_gemm python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
ls -la gpurun_out
