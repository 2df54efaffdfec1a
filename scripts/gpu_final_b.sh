# Round-end measurement, part B: full ncu captures of the dgrad and wgrad GEMMs
# (launch IDs from part A's pick10.txt, passed as arguments).
mkdir -p gpurun_out
P='python scripts/profile_step.py --steps 2'
cap() { timeout 900 ncu --set full --clock-control none --import-source on -s $2 -c 1 -o gpurun_out/prof_$1 $P > /dev/null 2>&1; echo "ncu $1 rc=$?"; }
cap gemm_dgrad $1
cap gemm_wgrad $2
du -sh gpurun_out
