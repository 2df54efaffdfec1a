#!/bin/bash
# round 2: ncu of the small-M GEMMs (engine vs cuBLAS), exported as CSV (reports stay on the box)
mkdir -p gpurun_out /tmp/ncu
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02f_build.log 2>&1
for shp in "128 4096 8192 bmn" "128 8192 4096" "2496 8192 4096"; do
  tag=$(echo $shp | tr ' ' '_')
  FI_GEMM_LOG=1 timeout 300 ncu --set full --clock-control none -k regex:"k_gemm|nvjet|gemm" -c 6 \
     -o /tmp/ncu/r02f_$tag python scripts/gemm_one.py $shp > gpurun_out/r02f_$tag.log 2>&1
  ncu -i /tmp/ncu/r02f_$tag.ncu-rep --page raw --csv > gpurun_out/r02f_${tag}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/r02f_$tag.ncu-rep --page details --csv > gpurun_out/r02f_${tag}_details.csv 2>/dev/null
done
ls -la gpurun_out/ | grep r02f
