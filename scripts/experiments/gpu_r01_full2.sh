# Full GPU pass: smoke, GPU tests, bench (ours + reference arm), launch list, ncu full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q --tb=short 2>&1 | tail -5
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json; tail -3 gpurun_out/bench_r01b.err
timeout 600 python bench.py --gemm-dtype fp32 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01b_fp32.json 2>&1; tail -c 400 gpurun_out/bench_r01b_fp32.json
timeout 600 python bench.py --config 5 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_r01b_cfg5.json 2>&1; tail -c 1500 gpurun_out/bench_r01b_cfg5.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_r01b_ref.json 2>&1; cat gpurun_out/bench_r01b_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_split_fwd -s 57 -c 1 -o gpurun_out/prof_split python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu split rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_bwd -s 58 -c 1 -o gpurun_out/prof_gather python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gather rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 99 -c 1 -o gpurun_out/prof_gemm_fwd python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 138 -c 1 -o gpurun_out/prof_gemm_dgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 158 -c 1 -o gpurun_out/prof_gemm_wgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
ls -la gpurun_out
