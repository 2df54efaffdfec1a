mkdir -p gpurun_out
P='python scripts/profile_step.py --steps 2'
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_gemm<.*\(bool\)0, \(bool\)0, \(int\)5' -s 58 -c 1 -o gpurun_out/prof_gemm_fwd $P > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_gemm<.*\(bool\)0, \(bool\)1, \(int\)6' -s 58 -c 1 -o gpurun_out/prof_gemm_dgrad $P > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_gemm<.*\(bool\)1, \(bool\)1, \(int\)3' -s 3 -c 1 -o gpurun_out/prof_gemm_wgrad $P > /dev/null 2>&1; echo rc=$?
ls gpurun_out
