echo "== old"; FI_LIB_PATH=build_ab/old.so timeout 300 python scripts/per_width.py 2>&1 | tail -45
echo "== new"; FI_GEMM_LOG=1 timeout 300 python scripts/per_width.py > gpurun_out/pw_new.txt 2>&1; tail -45 gpurun_out/pw_new.txt
