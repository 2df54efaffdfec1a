#!/bin/bash
# round 2: config-5 (|N| = 8192, B = 128) and tf32-mode evidence: bench lines + ncu metrics of
# the forward / dgrad / wgrad GEMMs (tensor-pipe utilisation, DRAM bytes, duration)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02c5_build.log 2>&1
timeout 900 python bench.py --config 5 --no-cpu-baseline > gpurun_out/r02c5_bench_cfg5.json 2> gpurun_out/r02c5_bench_cfg5.err
timeout 900 python bench.py --gemm-dtype tf32 --no-cpu-baseline > gpurun_out/r02c5_bench_tf32.json 2> gpurun_out/r02c5_bench_tf32.err
timeout 900 python bench.py --gemm-dtype fp32 --no-cpu-baseline > gpurun_out/r02c5_bench_fp32.json 2> gpurun_out/r02c5_bench_fp32.err
M="gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second,l1tex__m_xbar2l1tex_read_bytes.sum"
for cfg in "8192 128 40 bf16" "4096 64 40 tf32"; do
  set -- $cfg
  timeout 900 ncu --metrics $M --clock-control none --csv -k regex:"k_gemm|k_split|k_gather" \
    --log-file gpurun_out/r02c5_ncu_n$1_$4.csv python scripts/profile_step.py --n $1 --batch $2 --length $3 --dtype $4 --steps 2 > /dev/null 2>&1
  echo "ncu $cfg rc=$?"
done
ls -la gpurun_out | grep r02c5
