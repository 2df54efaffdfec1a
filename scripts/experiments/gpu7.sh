mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json; tail -3 gpurun_out/bench_r01.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 55 -c 1 -o gpurun_out/prof_split python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 58 -c 1 -o gpurun_out/prof_gather python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 98 -c 1 -o gpurun_out/prof_gemm_fwd python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 140 -c 1 -o gpurun_out/prof_gemm_dgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 158 -c 1 -o gpurun_out/prof_gemm_wgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
ls gpurun_out
