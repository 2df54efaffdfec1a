for cfg in "FI_GEMM_SK=0 FI_GEMM_BN=256" "FI_GEMM_SK=0 FI_GEMM_BN=128" "FI_GEMM_SK=0 FI_GEMM_BN=64" "FI_GEMM_SK=1 FI_GEMM_BN=256" "FI_GEMM_SK=1 FI_GEMM_BN=128"; do
echo "== $cfg"; env $cfg timeout 300 python scripts/gemm_micro.py
done
FI_GEMM_SK=1 FI_GEMM_BN=256 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemm -s 4 -c 1 python scripts/gemm_micro.py 2>&1 | grep -E "k_gemm|duration|bytes|hit|tensor" | tail -6
FI_GEMM_SK=0 FI_GEMM_BN=256 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:k_gemm -s 4 -c 1 python scripts/gemm_micro.py 2>&1 | grep -E "k_gemm|duration|bytes|hit|tensor" | tail -6
