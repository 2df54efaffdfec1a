mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json; tail -3 gpurun_out/bench_r01.err
timeout 600 python bench.py --steps 5 --warmup 3 --gemm-dtype fp32 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01_fp32.json 2>&1; tail -c 600 gpurun_out/bench_r01_fp32.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01_ref.json 2>&1; cat gpurun_out/bench_r01_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 55 -c 2 -o gpurun_out/prof_split python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 50 -c 2 -o gpurun_out/prof_gather python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 160 -c 2 -o gpurun_out/prof_gemm_wgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
ls gpurun_out
