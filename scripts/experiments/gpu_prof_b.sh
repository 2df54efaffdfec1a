mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 138 -c 1 -o gpurun_out/prof_gemm_dgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gemm -s 158 -c 1 -o gpurun_out/prof_gemm_wgrad python scripts/profile_step.py --steps 2 > /dev/null 2>&1; echo "ncu gemm rc=$?"
du -sh gpurun_out
