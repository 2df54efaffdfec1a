#!/bin/bash
# source-level (SASS) ncu view of the config-3 width-20 gather and split launches
mkdir -p gpurun_out /tmp/ncu
P='python scripts/profile_step.py --steps 2'
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/ncu/l.csv $P > /dev/null 2>&1
python scripts/pick_launches.py /tmp/ncu/l.csv 20 40 > /tmp/ncu/pick.txt; cat /tmp/ncu/pick.txt
for k in gather split; do
  id=$(awk -v k=$k '$1==k{print $2}' /tmp/ncu/pick.txt)
  timeout 900 ncu --set full --clock-control none --import-source on -s $id -c 1 -o /tmp/ncu/src_$k $P > /dev/null 2>&1
  ncu -i /tmp/ncu/src_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r02src_${k}_sass.csv 2>/dev/null
  ncu -i /tmp/ncu/src_$k.ncu-rep --page raw --csv > gpurun_out/r02src_${k}_raw.csv 2>/dev/null
done
ls -la gpurun_out/r02src*
