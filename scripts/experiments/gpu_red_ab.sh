bash scripts/gpu_pw_multi.sh head.so red.so > gpurun_out/red_ab.txt 2>&1
for us in 6 3; do echo "== red.so RED_US=$us" >> gpurun_out/red_ab.txt; FI_GEMM_RED_US=$us FI_LIB_PATH=build_ab/red.so timeout 300 python scripts/per_width.py 2>&1 | tail -45 >> gpurun_out/red_ab.txt; done
bash scripts/gpu_pw_multi.sh head.so red.so >> gpurun_out/red_ab.txt 2>&1
