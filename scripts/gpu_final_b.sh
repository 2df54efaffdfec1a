mkdir -p gpurun_out
SECONDS=0
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
echo "bench wall ${SECONDS}s"
python scripts/bj.py final < gpurun_out/bench_final.json
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 99 -c 1 -o gpurun_out/prof_gemm_fwd python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gemm<" -s 150 -c 1 -o gpurun_out/prof_gemm_dgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
du -sh gpurun_out
