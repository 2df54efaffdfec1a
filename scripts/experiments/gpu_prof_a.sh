mkdir -p gpurun_out
cp -f /dev/null gpurun_out/.keep
timeout 600 python bench.py --gemm-dtype fp32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01b_fp32.json 2>&1
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01b_cfg5.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 57 -c 1 -o gpurun_out/prof_split python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 58 -c 1 -o gpurun_out/prof_gather python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 99 -c 1 -o gpurun_out/prof_gemm_fwd python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
du -sh gpurun_out
